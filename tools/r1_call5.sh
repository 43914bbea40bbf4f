NVCC_APPEND_FLAGS=-DCDSP_DTRACE python paper_2511_06247_b200/build.py --force > /dev/null 2>&1; echo build=$?
timeout 300 python tools/decode_trace.py 262144 2>&1 | tail -16
timeout 300 python tools/decode_trace.py 32768 2>&1 | tail -6
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
