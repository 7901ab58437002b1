# absorbed: parity + q~ tile A/B
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k absorbed --timeout 300 2>&1 | tail -2
for bn in 128 256; do
  HC_QT_BN=$bn timeout 300 python bench.py --absorb --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('BN=$bn', round(d['ms_per_step'],3), round(d['kernels']['absorbed_hidden']['ms'],3))"
done
bash scripts/absorb_ncu.sh
