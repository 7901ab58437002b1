# fused-kernel raster A/B: n-tiles per n-major group (pairs of a wave sharing an A panel)
#   GROUP_LIST="2 4 6" NCU=1 bash scripts/group_ab.sh cfg4 cfg5:0.03125
for CFG in ${@:-cfg4 cfg5:0.03125}; do
for i in 1 2; do
for g in ${GROUP_LIST:-2 4 6}; do
  HC_GROUP_N=$g timeout 600 python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};k=d['kernels'];g=k.get('recon_gemm') or k.get('fused_step');print('$CFG group $g', round(d['ms_per_step'],3), round(d['step_ms_percentiles']['p50'],3), round(g['ms'],3), round(g.get('achieved') or 0), c.get('sm_mhz'), c.get('power_w'))"
done
done
done
if [ -n "$NCU" ]; then
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
for g in ${GROUP_LIST:-2 4 6}; do echo "ncu cfg4 group $g"; HC_GROUP_N=$g /usr/local/cuda/bin/ncu --metrics $M --clock-control none -k regex:fused -c 1 python bench.py --config cfg4 --profile-steps 1 2>&1 | grep -E "^    [a-z]"; done
fi
