O=gpurun_out/${TAG:-r4y}; mkdir -p $O
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_decode.py -q -x --timeout 300 -p no:cacheprovider > $O/pytest_dec.log 2>&1; echo "rc=$?" >> $O/pytest_dec.log; tail -n 3 $O/pytest_dec.log
bash tools/abdec.sh "-DCDSP_DEC_MERGE=1" "" > $O/ab.txt 2>&1; cat $O/ab.txt
NVCC_APPEND_FLAGS="-DCDSP_DTRACE" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
python tools/decode_trace.py > $O/trace.txt 2>&1
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
sed -n 1,10p $O/trace.txt
