O=gpurun_out/${TAG:-r4i}; mkdir -p $O
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
python tools/bench_decode.py --steps 20 > $O/decode.json 2>&1
./tools/read_rate.bin > $O/read.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_tma --launch-skip 6 --launch-count 1 -o $O/decode_tma python tools/bench_decode.py --steps 2 > $O/ncu.log 2>&1
tail -3 $O/ncu.log; cat $O/decode.json
