# Phase-2 strong scaling (bench.py --strong --split) on a 1-GPU box: 2 ranks on device 0
# over gloo (test hooks), with the rank-0 oracle check of the longest split request.
export HC_BENCH_ONE_GPU=1 HC_BENCH_BACKEND=gloo HC_BENCH_CHECK=1
for cfg in tiny cfg2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 \
    bench.py --gpus 2 --steps 3 --warmup 3 --config $cfg --strong --split > gpurun_out/split_$cfg.json 2> gpurun_out/split_$cfg.err
  echo "rc=$? cfg=$cfg"; tail -3 gpurun_out/split_$cfg.err | cut -c1-300; tail -1 gpurun_out/split_$cfg.json | cut -c1-900
done
HC_BENCH_CHECK=1 timeout 600 python bench.py --steps 3 --warmup 3 --config tiny --strong --split 2>&1 | tail -1 | cut -c1-600
