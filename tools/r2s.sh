O=gpurun_out/${TAG:-r2s}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fused.py -q -x --timeout 300 -p no:cacheprovider > $O/pytest_fast.log 2>&1; echo "rc=$?" >> $O/pytest_fast.log
tail -n 15 $O/pytest_fast.log
bash tools/ab.sh "-DCDSP_EPI_WARPS=1" "-DCDSP_EPI_WARPS=0" > $O/ab.txt 2>&1; cat $O/ab.txt
