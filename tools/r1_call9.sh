python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_multiproc.py -x -q 2>&1 | tail -30
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/bench_layers.py > gpurun_out/r01_layers.json 2> gpurun_out/layers.err; echo layers=$?; cat gpurun_out/r01_layers.json; tail -3 gpurun_out/layers.err
