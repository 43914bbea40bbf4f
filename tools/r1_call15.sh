#!/bin/bash
# persistent attn_tc (v9): parity, bench, loopback SP sweep
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_striped.py tests/test_gpu_layers.py -x -q 2>&1 | tail -5
for i in 1 2; do timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('BENCH', d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'])"; done
timeout 600 python tools/bench_interleave.py 2>&1 | tail -1
