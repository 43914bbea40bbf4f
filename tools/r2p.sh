O=gpurun_out/${TAG:-r2p}; mkdir -p $O
bash tools/ab.sh "-DCDSP_ALL_LANE_ARRIVE=1" "-DCDSP_ALL_LANE_ARRIVE=0" > $O/ab.txt 2>&1
cat $O/ab.txt
