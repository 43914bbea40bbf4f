#!/bin/bash
# Dev: same-box A/B of build-flag variants on the per-GPU ring proxy (tools/bench_rank_ring.py, split mode).
# usage: tools/ab_rank.sh "<flags A>" "<flags B>" ...   (SIZES=4,8 by default)
for round in 1 2; do
  for flags in "$@"; do
    NVCC_APPEND_FLAGS="$flags" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
    echo -n "[$flags] "
    python tools/bench_rank_ring.py --sizes ${SIZES:-4,8} --modes split --iters 8 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print({k:round(v['tflops_per_gpu']) for k,v in d['results'].items()})"
  done
done
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
