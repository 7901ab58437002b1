# Same-box A/B of two builds of libhc.so (ab/libhc_A.so, ab/libhc_B.so; untracked scratch).
#   bash scripts/lib_ab.sh cfg2 cfg4 ...
for CFG in ${@:-cfg2 cfg4}; do
for i in ${REPS:-1 2}; do
for v in A B; do
  cp ab/libhc_$v.so paper_2504_07494_b200/libhc.so
  timeout 600 python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};k=d['kernels'];g=k.get('recon_gemm') or k.get('fused_step') or k.get('attention');print('$CFG $v', round(d['ms_per_step'],3), round(d['step_ms_percentiles']['p50'],3), round(d['step_ms_percentiles']['p90'],3), round(g['ms'],3), round(g.get('achieved') or 0), c.get('sm_mhz'), c.get('power_w'))"
done
done
done
cp ab/libhc_B.so paper_2504_07494_b200/libhc.so
