#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over tools/sanitize_cases.py
O=gpurun_out/${TAG:-sanitize}; mkdir -p $O
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
timeout 300 python tools/sanitize_cases.py > $O/plain.log 2>&1; echo "rc=$?" >> $O/plain.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_cases.py > $O/$t.log 2>&1; echo "rc=$?" >> $O/$t.log
done
tail -n 4 $O/*.log
