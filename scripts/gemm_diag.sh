# Fused-kernel GEMM diagnostics (timing only; HC_DIAG_* give wrong outputs):
#   HC_DIAG_EPI=1 skip the attend epilogue math; HC_DIAG_BOX=1 128-row A boxes (as if dense);
#   HC_SYNC_W=0 partner lockstep off; HC_SYNC_W=2/32 window.
CFG=${1:-cfg4}
for i in 1 2; do
for env in "HC_X=0" "HC_DIAG_BOX=1" "HC_SYNC_W=0" "HC_SYNC_W=2" "HC_SYNC_W=32" "HC_DIAG_EPI=1 HC_DIAG_BOX=1"; do
  env $env timeout 600 python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};k=d['kernels'];g=k.get('recon_gemm') or k.get('fused_step');print('$CFG $env', round(d['ms_per_step'],3), round(g['ms'],3), round(g.get('achieved') or 0), c.get('sm_mhz'), c.get('power_w'))"
done
done
