set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -25
timeout 300 python tools/bench_decode.py > gpurun_out/bench_decode.json 2>&1; echo dec=$?; cat gpurun_out/bench_decode.json
timeout 300 python tools/bench_decode.py --ctx 32768 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_mma -s 24 -c 1 -o gpurun_out/decode_mma_full python tools/bench_decode.py --steps 1 > gpurun_out/ncu_dec.log 2>&1; echo ncu=$?
timeout 600 python -m pytest tests/test_gpu_ring.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -3
