#!/bin/bash
# 2-SM attn_tc: parity first, then speed
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -8
for i in 1 2; do timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('BENCH', d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'])"; done
CDSP_ATTN_1SM=1 timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('BENCH-1SM', d['value'], d['roofline']['achieved'])"
