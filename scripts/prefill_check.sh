# f3 prefill: parity (tcgen05 BK 64/128 + mma.sync attention) and the OPT-66B prefill bench A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill or recompute or rope_layer" --timeout 600 2>&1 | tail -2
HC_PREFILL_BK=128 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_layer and tc" --timeout 600 2>&1 | tail -2
for bk in 64 128; do
  for L in 512 2048 4096; do
    HC_PREFILL_BK=$bk timeout 600 python bench.py --mode prefill --prefill-len $L --prefill-reqs 8 --steps 10 --warmup 3 --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('bk=$bk L=$L', round(d['ms_per_step'],3), round(d['value']))"
  done
done
HC_PREFILL_BK=64 L=2048 bash scripts/prefill_ncu.sh
