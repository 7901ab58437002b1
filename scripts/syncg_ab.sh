# A/B of the A-panel sharing group (HC_SYNC_G): parity, crossover and cfg4 under sustained load
HC_SYNC_G=6 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "opt_shaped or fused or alternative_gemm or all_hidden or mixed_batch" --timeout 300 2>&1 | tail -2
for g in 2 6 4; do
  for h in 0.03125 0.0625; do
    HC_SYNC_G=$g timeout 600 python bench.py --config cfg5:$h --steps 300 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};print('G=$g h=$h', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), c.get('sm_mhz'))"
  done
  HC_SYNC_G=$g timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};print('G=$g cfg4', round(d['ms_per_step'],3), round(d['roofline']['achieved']), c.get('sm_mhz'))"
done
