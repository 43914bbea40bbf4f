#!/bin/bash
# Dev: same-box A/B of build-flag variants of the decode kernel (tools/bench_decode.py).
for round in 1 2; do
  for flags in "$@"; do
    NVCC_APPEND_FLAGS="$flags" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
    echo -n "[$flags] "
    python tools/bench_decode.py --steps 20 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['avg_launch_us'],1), round(d['step_us_all_ranks']/8,1))"
  done
done
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
