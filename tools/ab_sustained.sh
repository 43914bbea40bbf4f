#!/bin/bash
# Dev: sustained (power-capped) A/B of build-flag variants: each runs the bench attention
# back-to-back for $SECS seconds under nvidia-smi sampling (tools/clock_probe.py).
SECS=${SECS:-4}
for flags in "$@"; do
  NVCC_APPEND_FLAGS="$flags" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
  NVCC_APPEND_FLAGS="$flags" python tools/clock_probe.py $SECS 2>&1 | tail -1
  sleep 3
done
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
