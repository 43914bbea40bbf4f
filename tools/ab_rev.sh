#!/bin/bash
# Dev: same-box A/B of the working tree against an older attn_tc.cu (tools/old_attn_tc.cu.txt).
rm -rf /tmp/old_repo && cp -r . /tmp/old_repo && cp tools/old_attn_tc.cu.txt /tmp/old_repo/paper_2511_06247_b200/csrc/attn_tc.cu
(cd /tmp/old_repo && python paper_2511_06247_b200/build.py --force > /dev/null 2>&1)
python paper_2511_06247_b200/build.py > /dev/null 2>&1
for round in 1 2 3; do
  for d in . /tmp/old_repo; do
    echo -n "[$d] "
    (cd $d && python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'], end=' ')"
     python tools/bench_rank_ring.py --iters 5 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(' '.join(k+'='+str(round(v['tflops_per_gpu'])) for k,v in d['results'].items()))")
  done
done
