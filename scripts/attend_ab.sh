# fused reconstruct-and-attend epilogue: parity, then A/B vs the scratch path (HC_EPI_ATTEND=0)
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "not absorbed and not prefill and not ln" 2>&1 | tail -4
for env in "HC_EPI_ATTEND=1" "HC_EPI_ATTEND=0"; do
  env $env timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};k=d['kernels'];g=k.get('recon_gemm') or k.get('fused_step');print('$env cfg4', round(d['ms_per_step'],3), round(g['ms'],3), round(g['achieved']), c.get('sm_mhz'), c.get('power_w'))"
  for h in 0.03125 0.125; do
    env $env timeout 600 python bench.py --config cfg5:$h --steps 200 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};print('$env h=$h', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), c.get('sm_mhz'))"
  done
done
