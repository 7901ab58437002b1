# N>1 control path of bench.py on a 1-GPU box: 2 ranks on device 0 over gloo (test hook)
export HC_BENCH_ONE_GPU=1 HC_BENCH_BACKEND=gloo
for extra in "" "--strong" "--gather"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 5 --warmup 3 --config cfg2 $extra > gpurun_out/mr.json 2> gpurun_out/mr.err
  echo "rc=$? extra=$extra"; tail -2 gpurun_out/mr.err | cut -c1-300
  python -c "
import json;L=[l for l in open('gpurun_out/mr.json').read().splitlines() if l.startswith('{')];print(len(L), 'lines');d=json.loads(L[-1]);print(d['n_gpus'], round(d['ms_per_step'],3), round(d['value']), d['scaling'], d['config']['parallelism'], d['config'].get('output_gather'), d.get('e2e',{}).get('value'))"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --impl reference --gpus 2 --steps 2 --warmup 1 --config cfg2 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err
echo "ref rc=$?"; cat gpurun_out/mr_ref.json | cut -c1-300
