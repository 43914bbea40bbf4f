python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python tools/bench_decode.py > gpurun_out/r01_decode_bench.json 2>&1; echo dec=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_mma -s 24 -c 1 -o gpurun_out/decode_mma_full2 python tools/bench_decode.py --steps 1 > gpurun_out/ncu_dec.log 2>&1; echo ncu=$?
