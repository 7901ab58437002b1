# fused-kernel configuration A/B (HC_FUSED_CFG: GEMM stages / attention warps / attention
# stages, suffix 0 = q in registers): 342 default, 3420, 352 (5 attention warps, q in registers)
for CFG in ${@:-cfg5:0.015625 cfg5:0.03125 cfg5:0.0625 cfg4}; do
for i in 1 2; do
for c in ${CFG_LIST:-342 3420 352}; do
  HC_FUSED_CFG=$c timeout 600 python bench.py --config $CFG --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};p=d['step_ms_percentiles'];k=d['kernels'];g=k.get('recon_gemm') or k.get('fused_step');print('$CFG cfg $c', round(d['ms_per_step'],3), round(p['p50'],3), round(p['max'],3), round(g['ms'],3), c.get('sm_mhz'), c.get('power_w'))"
done
done
done
