#!/bin/bash
CDSP_KTRACE=1 python paper_2511_06247_b200/build.py --force > /dev/null 2>&1; echo build=$?
timeout 300 python tools/trace_units.py gpurun_out 2>&1 | grep -v Warn | head -14
python tools/an_tiles.py gpurun_out/trace_s1.bin
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
