#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, optional extra commands.  Outputs under gpurun_out/$TAG.
# usage (on the box): bash tools/gpu_run.sh TAG "<pytest selection or -m gpu>" [extra command ...]
TAG=${1:-run}; SEL=${2:-"-m gpu"}; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
if [ "$SEL" != "none" ]; then
  timeout 1500 python -m pytest tests $SEL -q --timeout 600 -p no:cacheprovider > $OUT/pytest.log 2>&1
  echo "pytest rc=$?" >> $OUT/pytest.log
  tail -5 $OUT/pytest.log
fi
for cmd in "$@"; do
  echo "== $cmd" >> $OUT/extra.log
  timeout 900 bash -c "$cmd" >> $OUT/extra.log 2>&1
  echo "rc=$?" >> $OUT/extra.log
done
tail -c 3000 $OUT/extra.log 2>/dev/null
