O=gpurun_out/${TAG:-r2j}; mkdir -p $O
CDSP_KTRACE=1 python paper_2511_06247_b200/build.py --force > /dev/null 2>&1 && timeout 600 python tools/trace_units.py $O > $O/trace.txt 2>&1
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
rm -f $O/*.bin; grep -E "==|per SM|fit loop|boundary|tail" $O/trace.txt
