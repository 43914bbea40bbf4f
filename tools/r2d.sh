O=gpurun_out/r2d; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for ord in 0 1; do CDSP_UNIT_ORDER=$ord timeout 600 python tools/bench_rank_ring.py --iters 5 --sizes 2,4,8 --modes fused > $O/rank_ring_order$ord.json 2>&1; done
timeout 600 python tools/bench_mem_kernels.py > $O/mem.json 2>&1
timeout 600 ncu --set full --clock-control none -k regex:store_append -s 0 -c 1 -o $O/mem_append python tools/bench_mem_kernels.py --iters 1 --only append > $O/ncu_append.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:row_copy -s 3 -c 1 -o $O/mem_gather python tools/bench_mem_kernels.py --iters 1 --only gather > $O/ncu_gather.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:lse_merge -s 3 -c 1 -o $O/mem_merge2 python tools/bench_mem_kernels.py --iters 1 --only merge2 > $O/ncu_merge2.log 2>&1
CDSP_KTRACE=1 python paper_2511_06247_b200/build.py --force > /dev/null 2>&1 && timeout 600 python tools/trace_units.py $O > $O/trace.txt 2>&1
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
rm -f $O/*.bin
tail -3 $O/pytest.log
