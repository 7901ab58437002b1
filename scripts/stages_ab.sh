# GEMM ring depth A/B: fused {GEMM stages, attention warps, attention stages} = 342 (default) / 422 / 412
for CFG in ${@:-cfg4 cfg2 cfg5:0.03125 cfg5:0.125}; do
for i in 1 2; do
for env in "HC_FUSED_CFG=342" "HC_FUSED_CFG=422" "HC_FUSED_CFG=412"; do
  env $env timeout 600 python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};k=d['kernels'];g=k.get('recon_gemm') or k.get('fused_step');print('$CFG $env', round(d['ms_per_step'],3), round(g['ms'],3), round(g.get('achieved') or 0), c.get('sm_mhz'), c.get('power_w'))"
done
done
done
