#!/bin/bash
# Dev: same-box A/B of build-flag variants: s=1 bench kernel TF/s and loopback SP sweep (zigzag).
# usage: tools/ab2.sh "<flags A>" "<flags B>" ...
for round in 1 2; do
  for flags in "$@"; do
    NVCC_APPEND_FLAGS="$flags" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
    echo -n "[$flags] s1: "
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'], end=' ')"
    python tools/bench_interleave.py --zigzag-only 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(' '.join(k+'='+str(round(v['tflops'])) for k,v in d['results'].items()))"
  done
done
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
