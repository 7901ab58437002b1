# fused step kernel vs the two-kernel path (stand-alone GEMM with the attend epilogue, then the KV attention kernel)
for CFG in ${@:-cfg5:0.125 cfg5:0.25 cfg4}; do
for i in 1 2 3; do
for f in 1 0; do
  HC_FUSED=$f timeout 600 python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};k=d['kernels'];g=k.get('recon_gemm') or k.get('fused_step');print('$CFG fused=$f', round(d['ms_per_step'],3), round(d['step_ms_percentiles']['p50'],3), round(d['step_ms_percentiles']['p90'],3), round(g['ms'],3), round(k['attention']['ms'],3), c.get('sm_mhz'), c.get('power_w'))"
done
done
done
