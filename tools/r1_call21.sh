#!/bin/bash
for dbg in none 0; do
  if [ $dbg = none ]; then extra=""; else extra="-DCDSP_DBG_SOFTMAX=$dbg"; fi
  CDSP_KTRACE=1 CDSP_NVCC_EXTRA="$extra" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
  echo "== PAIR DBG $dbg"
  timeout 300 python tools/trace_units.py gpurun_out 2>&1 | grep -v Warn | head -16
  python tools/an_tiles.py gpurun_out/trace_s1.bin
done
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
