# Timing diagnostic: how much of the fused step is the EPI_ATTEND epilogue (serialised with
# the next tile's mainloop: one 512-column accumulator).  HC_DIAG_EPI=1 skips the epilogue
# math (outputs are wrong; timing only).
CFG=${1:-cfg4}
for i in 1 2; do
for env in "HC_DIAG_EPI=0" "HC_DIAG_EPI=1" "HC_DIAG_EPI=2"; do
  env $env timeout 600 python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};k=d['kernels'];g=k.get('recon_gemm') or k.get('fused_step');print('$CFG $env', round(d['ms_per_step'],3), round(g['ms'],3), round(g.get('achieved') or 0), c.get('sm_mhz'), c.get('power_w'))"
done
done
