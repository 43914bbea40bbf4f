set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q 2>&1 | tail -15
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv -lms 50 > gpurun_out/clocks_long.csv &
CK=$!
timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_long.json 2>&1; echo long=$?
kill $CK
cat gpurun_out/bench_long.json
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e; echo short=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 -o gpurun_out/attn_full_v8 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_scatter -s 3 -c 1 -o gpurun_out/paged_full_v8 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full2.log 2>&1; echo ncufull2=$?
