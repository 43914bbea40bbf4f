#!/bin/bash
# Round-2 evidence (one gpurun call, outputs under gpurun_out/$TAG): ncu launch list of bench.py
# (s=1), --set full captures of the s=1 attention, the fused rank launches at s=2/4/8, the weak
# N=1 launch and every HBM-bound kernel; JSON timings of the memory kernels, decode and the
# per-GPU ring proxy.  Summarise here with tools/ncu_summary.py into profiles/.
O=gpurun_out/${TAG:-profiles}; mkdir -p $O
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 1 -c 1 -o $O/attn_s1 python tools/ncu_one_attn.py > $O/ncu_attn.log 2>&1
for s in 2 4 8; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 1 -c 1 -o $O/fused_s${s}_r0 \
    python tools/ncu_fused_rank.py --s $s --r 0 --split > $O/ncu_fused_s${s}.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 -o $O/weak_s1 \
  python bench.py --weak --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_weak.log 2>&1
for spec in "merge2:lse_merge:3" "merge8:lse_merge:3" "gather:row_copy:3" "scatter:row_copy:3" "append:store_append:0" "paged:paged_scatter:3"; do
  IFS=: read n k sk <<< "$spec"
  timeout 600 ncu --set full --clock-control none -k regex:$k -s $sk -c 1 -o $O/mem_$n python tools/bench_mem_kernels.py --iters 1 --only $n > $O/ncu_mem_$n.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_tma --launch-skip 6 --launch-count 1 -o $O/decode_tma python tools/bench_decode.py --steps 2 > $O/ncu_decode.log 2>&1
timeout 600 python tools/bench_mem_kernels.py > $O/mem.json 2>&1
timeout 600 python tools/bench_decode.py --steps 20 > $O/decode.json 2>&1
timeout 900 python tools/bench_rank_ring.py --iters 10 > $O/rank_ring.json 2>&1
./tools/read_rate.bin > $O/read_ceiling.txt 2>&1 || true
ls $O
