#!/bin/bash
# Dev: time the attention kernel for several FMA-pipe exp2 fractions (CDSP_EMU_MASK).
# usage: tools/sweep_emu.sh [mask ...]   (default: 0x00 0x02 0x22 0x52)
masks="${@:-0x00 0x02 0x22 0x52}"
for mask in $masks; do
  NVCC_APPEND_FLAGS="-DCDSP_EMU_MASK=$mask" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
  echo -n "mask=$mask "
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['roofline']['achieved'], d['roofline']['avg_launch_ms'])"
done
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
