#!/bin/bash
# Dev: same-box A/B of build-flag variants of the attention kernel.
# usage: tools/ab.sh "<flags A>" "<flags B>" ...   (each variant timed twice, interleaved)
for round in 1 2; do
  for flags in "$@"; do
    NVCC_APPEND_FLAGS="$flags" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
    echo -n "[$flags] "
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['roofline']['achieved'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
  done
done
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
