O=gpurun_out/${TAG:-r4x}; mkdir -p $O
python paper_2511_06247_b200/build.py --force > /dev/null 2>&1
export CDSP_BENCH_DEVICE=0 CUDA_DEVICE_MAX_CONNECTIONS=32
for args in "--gpus 4 --steps 2 --warmup 1 --no-e2e" "--gpus 8 --steps 2 --warmup 1 --no-e2e"; do
  n=$(echo $args | awk '{print $2}')
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 bench.py $args > $O/out_$n.txt 2> $O/err_$n.txt
  echo "N=$n rc=$?" >> $O/summary.txt
  grep '^{' $O/out_$n.txt | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['n_gpus'], d['config']['sp'], round(d['value']), d['gpu_launches'], d['ring'])" >> $O/summary.txt 2>&1
done
cat $O/summary.txt; tail -3 $O/err_8.txt
