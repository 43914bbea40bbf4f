O=gpurun_out/${TAG:-r4q}; mkdir -p $O
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_prefill_transfer.py tests/test_gpu_multiproc.py -q -x --timeout 300 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; tail -n 5 $O/pytest.log
for i in 1 2; do
  python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['roofline']['achieved']), d['gpu_launches'], d['clocks'].get('sm_min_mhz'))" >> $O/ab.txt
done
cat $O/ab.txt
