O=gpurun_out/${TAG:-r2h}; mkdir -p $O
for v in "0 " "0 --split" "7 --split"; do set -- $v; n=r$1${2:+_split};
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 1 -c 1 -o $O/fused_s8_$n python tools/ncu_fused_rank.py --s 8 --r $v > $O/ncu_$n.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -n 3 $O/pytest.log
