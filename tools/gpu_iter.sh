#!/bin/bash
# Dev: one GPU iteration on the attention kernel: parity tests, bench x2, KTRACE timeline.
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -3
for i in 1 2; do
  timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('BENCH', d['value'], d['roofline']['achieved'], d['roofline']['avg_launch_ms'], d['clocks'])"
done
if [ -n "$TRACE" ]; then
  CDSP_KTRACE=1 python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
  CDSP_TRACE=gpurun_out/$TRACE python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo trace=$?
  python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
fi
