O=gpurun_out/${TAG:-r2n}; mkdir -p $O
timeout 300 python tools/sanitize_cases.py > $O/plain.log 2>&1; echo "rc=$?" >> $O/plain.log
for t in racecheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_cases.py > $O/$t.log 2>&1; echo "rc=$?" >> $O/$t.log
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench.json 2>&1
timeout 600 python tools/bench_rank_ring.py --iters 5 --sizes 1,2,4,8 --modes split,stepwise > $O/rr.json 2>&1
timeout 1500 python -m pytest tests/test_gpu_fused.py tests/test_gpu_kernels.py tests/test_gpu_ring.py -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -n 3 $O/*.log; python -c "
import json;d=json.load(open('$O/rr.json'));print({k:(round(v['tflops_per_gpu']),round(v['rank_ms_max'],3),round(v['rank_ms_min'],3)) for k,v in d['results'].items()})
d=json.load(open('$O/bench.json'));print(d['value'],d['roofline']['achieved'],d['roofline']['frac'])"
