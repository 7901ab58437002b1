# A/B of the absorbed score pipeline depth (HC_SCORE_ST) on cfg4 + parity
mkdir -p gpurun_out
for st in 3 2; do
  HC_SCORE_ST=$st timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "absorbed_mixed or absorbed_hidden_only" --timeout 300 2>&1 | tail -1
  HC_SCORE_ST=$st timeout 300 python bench.py --absorb --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('st=$st', round(d['ms_per_step'],3), round(d['kernels']['absorbed_hidden']['ms'],3), round(d['kernels']['attention']['ms'],3))"
done
