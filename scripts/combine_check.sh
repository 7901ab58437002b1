timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "not prefill and not ln" 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused|combine" --csv --log-file gpurun_out/comb.csv python bench.py --profile-steps 2 > /dev/null 2>&1
grep combine gpurun_out/comb.csv | cut -d, -f5,15 | tail -2
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);c=d['clocks'] or {};print('cfg4', round(d['ms_per_step'],3), d['kernels']['combine'], c.get('sm_mhz'))"
