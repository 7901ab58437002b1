# crossover (cfg5 h=1/32): fused-kernel ncu summary + configuration A/B (sustained)
mkdir -p gpurun_out/xo
timeout 900 ncu --set full --clock-control none -k regex:"fused_step" -c 1 -o gpurun_out/xo/fused_h32 python bench.py --config cfg5:0.03125 --profile-steps 1 > /dev/null 2>&1
ncu -i gpurun_out/xo/fused_h32.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); hdr,units,vals=rows[0],rows[1],rows[2]
for w in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed','sm__cycles_elapsed.avg.per_second','lts__t_sector_hit_rate.pct']:
  for i,h in enumerate(hdr):
    if h==w: print(w, vals[i], units[i])
"
for cfg in 342 243 262; do
  for h in 0.03125 0.0625; do
    HC_FUSED_CFG=$cfg timeout 600 python bench.py --config cfg5:$h --steps 200 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};print('cfg=$cfg h=$h', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), c.get('sm_mhz'))"
  done
done
