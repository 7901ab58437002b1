# split-release accumulator: timing on cfg2 / cfg4 (+ epilogue-skip diagnostic for the bound)
for CFG in ${@:-cfg2 cfg4}; do
for i in 1 2; do
for env in "HC_SYNC_W=0 HC_SPLIT_REL=0" "HC_SYNC_W=0 HC_SPLIT_REL=1"; do
  env $env timeout 600 python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};k=d['kernels'];g=k.get('recon_gemm') or k.get('fused_step');print('$CFG $env', round(d['ms_per_step'],3), round(d['step_ms_percentiles']['p50'],3), round(g['ms'],3), round(g.get('achieved') or 0), c.get('sm_mhz'), c.get('power_w'))"
done
done
done
