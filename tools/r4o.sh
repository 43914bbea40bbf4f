O=gpurun_out/${TAG:-r4o}; mkdir -p $O
for i in 1 2; do
for f in "" "-DCDSP_DEC_HINT=1" "-DCDSP_DEC_NOWAIT=1"; do
  NVCC_APPEND_FLAGS="$f" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
  for e in "CDSP_BENCH_SEPARATE_XFER=1" "X=1"; do
    if [ "$f" != "" ] && [ "$e" != "X=1" ]; then continue; fi
    echo -n "[$f $e] " >> $O/ab.txt
    env $e python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['value']), round(d['roofline']['achieved']), d['gpu_launches'], d['clocks'].get('sm_min_mhz'))" >> $O/ab.txt
  done
done; done
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
cat $O/ab.txt
