#!/bin/bash
# Dev: parity subset (attention kernels + fused ring) under a build flag, then same-box A/B
# (attention s=1 via tools/ab.sh, ring proxy via tools/ab_rank.sh) against the default.
# usage: FLAG="-DCDSP_X=1" TAG=x bash tools/ab_flag.sh
O=gpurun_out/${TAG:-flag}; mkdir -p $O
NVCC_APPEND_FLAGS="$FLAG" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fused.py -q -x --timeout 300 -p no:cacheprovider -k "not pacing" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; tail -n 2 $O/pytest.log
bash tools/ab.sh "" "$FLAG"
SIZES=8 bash tools/ab_rank.sh "" "$FLAG"
