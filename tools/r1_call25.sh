#!/bin/bash
# which softmax activity slows the 2-SM tensor pipe? (debug builds; results garbage)
for dbg in none 0 1 2 3; do
  if [ $dbg = none ]; then extra=""; else extra="-DCDSP_DBG_SOFTMAX=$dbg"; fi
  CDSP_KTRACE=1 NVCC_APPEND_FLAGS="$extra" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
  echo "== DBG $dbg"
  timeout 300 python tools/trace_units.py gpurun_out 2>&1 | grep -E "span|PV issue period" | head -2
done
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
