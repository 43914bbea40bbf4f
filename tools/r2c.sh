O=gpurun_out/r2c; mkdir -p $O
bash tools/ab.sh "-DCDSP_SUM_ROUNDED=1" "-DCDSP_SUM_ROUNDED=0" > $O/ab_sum.txt 2>&1
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
timeout 600 python tools/diag_precision.py > $O/diag.json 2>&1
timeout 600 python tools/bench_mem_kernels.py > $O/mem.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log; cat $O/ab_sum.txt
