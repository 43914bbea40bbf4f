python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_striped.py -x -q 2>&1 | tail -30
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/bench_interleave.py > gpurun_out/r01_interleave.json 2> gpurun_out/il.err; echo il=$?; cat gpurun_out/r01_interleave.json; tail -3 gpurun_out/il.err
timeout 400 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('BENCH', d['value'], d['roofline']['achieved'], d['roofline']['frac'])"
