O=gpurun_out/${TAG:-r4l}; mkdir -p $O
for f in "" "-DCDSP_EMU_MASK=0" "-DCDSP_EMU_MASK=0x0A"; do
  NVCC_APPEND_FLAGS="$f" python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
  for i in 1 2; do echo -n "[$f] " >> $O/sus.txt; python tools/sustain_probe.py >> $O/sus.txt 2>&1; done
done
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
cat $O/sus.txt
