O=gpurun_out/${TAG:-r2w}; mkdir -p $O
NVCC_APPEND_FLAGS="-DCDSP_NGROUPS=3 -DCDSP_EPI_WARPS=0" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 120 -p no:cacheprovider -k "causal_attention_all_rows or block_with_history" > $O/pytest_ng3.log 2>&1; echo "rc=$?" >> $O/pytest_ng3.log; tail -n 2 $O/pytest_ng3.log
bash tools/ab.sh "-DCDSP_EPI_WARPS=0" "-DCDSP_NGROUPS=3 -DCDSP_EPI_WARPS=0" "-DCDSP_NGROUPS=3 -DCDSP_EPI_WARPS=0 -DCDSP_FULL_ROW=0" "-DCDSP_EPI_WARPS=1" > $O/ab.txt 2>&1; cat $O/ab.txt
