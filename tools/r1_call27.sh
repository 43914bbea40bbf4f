#!/bin/bash
# round-1 measurement pass for attn_tc v11 (2-SM persistent, final round-1 pass)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
for i in 1 2; do timeout 400 python bench.py > gpurun_out/bench_v11_$i.json 2> gpurun_out/bench_v11_$i.err; echo bench=$?; cat gpurun_out/bench_v11_$i.json; done
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_v11.json 2>/dev/null; echo ref=$?; cat gpurun_out/bench_ref_v11.json
timeout 300 python bench.py --steps 300 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_v11_long.json 2>/dev/null; echo long=$?; cat gpurun_out/bench_v11_long.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v11.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1; echo ncu_list=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc --launch-skip 1 --launch-count 1 -o gpurun_out/attn_v11 python tools/ncu_one_attn.py > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
timeout 300 python tools/bench_rank_ring.py > gpurun_out/rank_ring_v11.json 2>/dev/null; cat gpurun_out/rank_ring_v11.json
timeout 600 python tools/bench_interleave.py > gpurun_out/interleave_v11.json 2>/dev/null; cat gpurun_out/interleave_v11.json
timeout 600 python tools/bench_layers.py > gpurun_out/layers_v11.json 2>/dev/null; cat gpurun_out/layers_v11.json
