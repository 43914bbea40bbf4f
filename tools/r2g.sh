O=gpurun_out/${TAG:-r2g}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_ring.py -q --timeout 600 -p no:cacheprovider -x > $O/pytest_fast.log 2>&1; echo "rc=$?" >> $O/pytest_fast.log
timeout 600 python tools/bench_rank_ring.py --iters 5 --sizes 1,2,4,8 --modes split,fused,stepwise > $O/rank_ring.json 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench.json 2>&1
tail -n 3 $O/pytest_fast.log; cat $O/rank_ring.json; python -c "import json;d=json.load(open('$O/bench.json'));print(d['value'],d['roofline']['achieved'],d['roofline']['frac'])"
