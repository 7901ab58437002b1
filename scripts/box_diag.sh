# A-operand gather diagnostic (timing only, wrong outputs): 16-row boxes from the block table
# (default) vs 16-row boxes over contiguous rows (HC_DIAG_EPI=3) vs one 128-row box (HC_DIAG_BOX=1)
for CFG in ${@:-cfg2 cfg4}; do
for i in 1 2; do
for env in "HC_X=0" "HC_DIAG_EPI=3" "HC_DIAG_BOX=1"; do
  env $env timeout 600 python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};k=d['kernels'];g=k.get('recon_gemm') or k.get('fused_step');print('$CFG $env', round(d['ms_per_step'],3), round(d['step_ms_percentiles']['p50'],3), round(g['ms'],3), round(g.get('achieved') or 0), c.get('sm_mhz'), c.get('power_w'))"
done
done
done
