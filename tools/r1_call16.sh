#!/bin/bash
CDSP_KTRACE=1 python paper_2511_06247_b200/build.py --force > /dev/null 2>&1; echo build=$?
timeout 300 python tools/trace_units.py gpurun_out 2>&1 | tail -40
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
