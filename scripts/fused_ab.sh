# fused-kernel configuration A/B at the crossover, sustained load (300 steps)
for cfg in 342 243 262 333; do
  for h in 0.03125 0.0625 0.125; do
    steps=$(python -c "print(300 if $h <= 0.0625 else 100)")
    HC_FUSED_CFG=$cfg timeout 600 python bench.py --config cfg5:$h --steps $steps --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};print('cfg=$cfg h=$h', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), c.get('sm_mhz'))"
  done
done
