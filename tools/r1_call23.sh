#!/bin/bash
# compact tile list + m(n) published before the exponentials; FMA-emulated exp fraction sweep
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -3
for mask in 0x02 0x22 0x26 0x66; do
  CDSP_NVCC_EXTRA="-DCDSP_EMU_MASK=$mask" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
  for i in 1 2; do timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('BENCH mask=$mask', round(d['value'],1), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
done
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
