#!/bin/bash
# One gpurun call: build, every GPU test, smoke, the default bench line and its ncu launch list
# (outputs under gpurun_out/$TAG).
O=gpurun_out/${TAG:-validate}; mkdir -p $O
python paper_2511_06247_b200/build.py --force > $O/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 2000 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -4 $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -3 $O/smoke.log
python bench.py > $O/bench.json 2> $O/bench.err; cat $O/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_bench.log 2>&1
echo "ncu rc=$?"
