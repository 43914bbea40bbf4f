#!/bin/bash
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc --launch-skip 1 --launch-count 1 -o gpurun_out/attn_pair python tools/ncu_one_attn.py > gpurun_out/ncu22.log 2>&1
echo ncu=$?
ncu -i gpurun_out/attn_pair.ncu-rep --page raw --csv > gpurun_out/attn_pair_raw.csv 2>/dev/null
ncu -i gpurun_out/attn_pair.ncu-rep --page source --csv --print-source cuda > gpurun_out/attn_pair_src.csv 2>/dev/null
ls -la gpurun_out/ | head
