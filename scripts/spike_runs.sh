# repeated short bench runs: mean vs p50 vs max step time (host/driver stalls show as max >> p50)
for CFG in ${@:-cfg4 cfg5:0.125}; do
for i in 1 2 3 4 5; do
  timeout 600 python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};p=d['step_ms_percentiles'];print('$CFG', round(d['ms_per_step'],3), round(p['p50'],3), round(p['p90'],3), round(p['max'],3), p.get('max_step'), c.get('sm_mhz'), c.get('samples'))"
done
done
