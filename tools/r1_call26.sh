#!/bin/bash
# a7 paged scatter grid cap vs the concurrent attention (bench step) and the scatter alone
timeout 600 python -m pytest tests/test_gpu_decode.py tests/test_gpu_fullsize.py -x -q -k "transfer or paged or M4" 2>&1 | tail -2
for cap in 16 8 32 100000; do
  for i in 1 2; do
    CDSP_SCATTER_CTAS=$cap timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('cap=$cap', 'step', round(d['value'],1), 'attn', round(d['roofline']['achieved'],1), d['ms_per_step'])"
  done
done
