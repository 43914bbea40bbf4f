CDSP_KTRACE=1 python paper_2511_06247_b200/build.py --force > /dev/null 2>&1; echo build=$?
timeout 300 python tools/trace_ring_step.py gpurun_out 2>&1 | grep -E "==|->|overhead|span"
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ring.py tests/test_gpu_striped.py -x -q 2>&1 | tail -2
for i in 1 2; do timeout 400 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('BENCH', d['value'], d['roofline']['achieved'], d['roofline']['frac'])"; done
timeout 600 python tools/bench_interleave.py 2>&1 | tail -1
