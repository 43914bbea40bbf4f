O=gpurun_out/${TAG:-r2f}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_ring.py -q --timeout 600 -p no:cacheprovider -x > $O/pytest_fast.log 2>&1; echo "rc=$?" >> $O/pytest_fast.log
timeout 600 python tools/bench_rank_ring.py --iters 5 --sizes 2,4,8 --modes split,fused > $O/rank_ring.json 2>&1
CDSP_KTRACE=1 python paper_2511_06247_b200/build.py --force > /dev/null 2>&1 && timeout 600 python tools/trace_units.py $O > $O/trace.txt 2>&1
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
rm -f $O/*.bin

tail -n 3 $O/pytest_fast.log; tail -n 3 $O/pytest.log; cat $O/rank_ring.json
