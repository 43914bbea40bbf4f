# Round-2 evidence: ncu launch list of bench.py (s=1), one --set full capture of the s=1 attention,
# fused s=8 ring launches (ranks 0 and 7, split scratch), every HBM-bound kernel; timings.
O=gpurun_out/${TAG:-r2y}; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file $O/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 1 -c 1 -o $O/attn_s1 python tools/ncu_one_attn.py > $O/ncu_attn.log 2>&1
for r in 0 7; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 1 -c 1 -o $O/fused_s8_r${r} python tools/ncu_fused_rank.py --s 8 --r $r --split > $O/ncu_fused_r$r.log 2>&1; done
for spec in "merge2:lse_merge:3" "merge8:lse_merge:3" "gather:row_copy:3" "scatter:row_copy:3" "append:store_append:0" "paged:paged_scatter:3"; do
  IFS=: read n k sk <<< "$spec"
  timeout 600 ncu --set full --clock-control none -k regex:$k -s $sk -c 1 -o $O/mem_$n python tools/bench_mem_kernels.py --iters 1 --only $n > $O/ncu_mem_$n.log 2>&1
done
timeout 600 python tools/bench_mem_kernels.py > $O/mem.json 2>&1
timeout 600 python tools/bench_decode.py > $O/decode.json 2>&1
timeout 900 python tools/bench_rank_ring.py --iters 5 --per 1 > $O/rank_ring.json 2>&1
ls $O
