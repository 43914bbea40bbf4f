O=gpurun_out/r2b; mkdir -p $O
timeout 600 python tools/diag_precision.py > $O/diag.json 2>&1
for r in 0 7; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 1 -c 1 -o $O/fused_s8_r$r python tools/ncu_fused_rank.py --s 8 --r $r > $O/ncu_fused_r$r.log 2>&1
done
timeout 600 python tools/bench_mem_kernels.py > $O/mem.json 2>&1
for spec in "merge2:lse_merge" "merge8:lse_merge" "gather:row_copy" "scatter:row_copy" "append:store_append" "paged:paged_scatter"; do
  n=${spec%%:*}; k=${spec##*:}
  timeout 600 ncu --set full --clock-control none -k regex:$k -s 3 -c 1 -o $O/mem_$n python tools/bench_mem_kernels.py --iters 1 --only $n > $O/ncu_mem_$n.log 2>&1
done
timeout 600 python tools/bench_rank_ring.py --iters 5 --sizes 8 --modes fused > $O/rank_ring_s8.json 2>&1
ls -la $O
