O=gpurun_out/${TAG:-r2i}; mkdir -p $O
for pol in 0 1; do
NVCC_APPEND_FLAGS="-DCDSP_KV_POLICY=$pol" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:attn_tc -s 1 -c 1 python tools/ncu_fused_rank.py --s 8 --r 0 --split > $O/ncu_pol$pol.log 2>&1
timeout 600 python tools/bench_rank_ring.py --iters 5 --sizes 1,8 --modes split > $O/rank_ring_pol$pol.json 2>&1
done
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
grep -E "dram__|lts__|gpu__time" $O/ncu_pol*.log; cat $O/rank_ring_pol*.json
