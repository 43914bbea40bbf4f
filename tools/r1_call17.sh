#!/bin/bash
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc --launch-skip 1 --launch-count 1 -o gpurun_out/attn_v9 python tools/ncu_one_attn.py > gpurun_out/ncu17.log 2>&1
echo ncu=$?
ncu -i gpurun_out/attn_v9.ncu-rep --page raw --csv > gpurun_out/attn_v9_raw.csv 2>/dev/null
ncu -i gpurun_out/attn_v9.ncu-rep --page details --csv > gpurun_out/attn_v9_details.csv 2>/dev/null
ls -la gpurun_out/
