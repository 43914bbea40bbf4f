O=gpurun_out/${TAG:-r2x}; mkdir -p $O
NVCC_APPEND_FLAGS="-DCDSP_COLSPLIT=1" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 120 -p no:cacheprovider -k "causal_attention_all_rows or block_with_history" > $O/pytest_cs.log 2>&1; echo "rc=$?" >> $O/pytest_cs.log; tail -n 3 $O/pytest_cs.log
timeout 400 python -m pytest tests/test_gpu_fused.py -q -x --timeout 120 -p no:cacheprovider > $O/pytest_cs_fused.log 2>&1; echo "rc=$?" >> $O/pytest_cs_fused.log; tail -n 3 $O/pytest_cs_fused.log
bash tools/ab.sh "" "-DCDSP_COLSPLIT=1" > $O/ab.txt 2>&1; cat $O/ab.txt
