python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -3
timeout 300 python tools/bench_decode.py 2>&1 | cut -c1-330
NVCC_APPEND_FLAGS=-DCDSP_DTRACE python paper_2511_06247_b200/build.py --force > /dev/null 2>&1; echo build=$?
timeout 300 python tools/decode_trace.py 262144 2>&1 | tail -8
timeout 300 python tools/decode_trace.py 32768 2>&1 | tail -8
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
