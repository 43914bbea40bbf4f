O=gpurun_out/${TAG:-r2k}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused.py -q --timeout 600 -p no:cacheprovider -x > $O/pytest_fast.log 2>&1; echo "rc=$?" >> $O/pytest_fast.log
for sp in 0 1 2; do CDSP_SPLIT=$sp timeout 600 python tools/bench_rank_ring.py --iters 5 --sizes 2,4,8 --modes split > $O/rank_ring_split$sp.json 2>&1; done
CDSP_KTRACE=1 python paper_2511_06247_b200/build.py --force > /dev/null 2>&1 && timeout 600 python tools/trace_units.py $O > $O/trace.txt 2>&1
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
rm -f $O/*.bin; tail -n 2 $O/pytest_fast.log; grep -E "==|per SM" $O/trace.txt; for sp in 0 1 2; do python -c "
import json;d=json.load(open('$O/rank_ring_split$sp.json'));print($sp, {k:(round(v['tflops_per_gpu']),round(v['rank_ms_max'],3),round(v['rank_ms_min'],3)) for k,v in d['results'].items()})"; done
