#!/bin/bash
# Context numbers: installed libraries' causal prefill attention vs ours on the s = 1 bench
# workload (tools/bench_library_attn.py), each backend in its own process with a time limit.
O=gpurun_out/${TAG:-libattn}; mkdir -p $O
python paper_2511_06247_b200/build.py > $O/build.log 2>&1
for rep in 1 2; do
for b in ours cudnn flash2 fi_fa2; do  # (flashinfer 0.6.11 single_prefill has no cutlass / trtllm-gen backend)
  timeout ${LIBT:-900} python tools/bench_library_attn.py --backend $b "$@" >> $O/lib.jsonl 2>> $O/lib.err || echo "{\"backend\": \"$b\", \"error\": \"rc=$?\"}" >> $O/lib.jsonl
done
done
cat $O/lib.jsonl
