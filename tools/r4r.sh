# ncu --set full of the dominant attention launch of more bench configurations (roofline.traffic keys)
O=gpurun_out/${TAG:-r4r}; mkdir -p $O
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
for s in 2 4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 1 -c 1 -o $O/ring_s${s} \
    python tools/ncu_fused_rank.py --s $s --r 0 --split > $O/ncu_s${s}.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 -o $O/weak_s1 \
  python bench.py --weak --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_weak.log 2>&1
ls -la $O; tail -2 $O/*.log
