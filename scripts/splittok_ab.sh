# KV split size A/B (bench.py --split-tokens; 0 = auto, 256 tokens at these sizes)
for CFG in ${@:-cfg5:0.03125 cfg5:0.0 cfg4}; do
for i in 1 2; do
for st in 0 512 1024; do
  timeout 600 python bench.py --config $CFG --split-tokens $st --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-graph 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};p=d['step_ms_percentiles'];k=d['kernels'];print('$CFG split $st', round(d['ms_per_step'],3), round(p['p50'],3), round(k['combine']['ms'],3), c.get('sm_mhz'))"
done
done
done
