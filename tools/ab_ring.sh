for round in 1 2; do
  for flags in "" "-DCDSP_EPI_WIDE=0"; do
    NVCC_APPEND_FLAGS="$flags" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
    echo -n "[$flags] "
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['roofline']['achieved'],1), end=' ')"
    python tools/bench_rank_ring.py --iters 5 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(' '.join(k+'='+str(round(v['tflops_per_gpu'])) for k,v in d['results'].items()))"
  done
done
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
