# same-box A/B: current tree vs old_tree (previous commit), cfg4, alternating
for i in 1 2; do
  timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};print('new', round(d['ms_per_step'],3), round(d['roofline']['achieved']), c.get('sm_mhz'))"
  (cd old_tree && timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};print('old', round(d['ms_per_step'],3), round(d['roofline']['achieved']), c.get('sm_mhz'))")
done
