# pair-tile width A/B on cfg4 (two-kernel path): 256x512 (NSUB 2, one accumulator) vs 256x256 (NSUB 1, double-buffered)
for i in 1 2; do
for env in "HC_FUSED=0" "HC_FUSED=0 HC_TC_NSUB=1" "HC_FUSED=1"; do
  env $env timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};k=d['kernels'];g=k.get('recon_gemm') or k.get('fused_step');print('$env', round(d['ms_per_step'],3), round(g['ms'],3), round(g['achieved']), c.get('sm_mhz'), c.get('power_w'))"
done
done
