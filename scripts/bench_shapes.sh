# bench lines for the OPT-13B (cfg2) and OPT-30B (cfg3, planner-assigned modes) layer shapes
mkdir -p gpurun_out/shapes
for c in cfg2 cfg3; do
  timeout 600 python bench.py --config $c --steps 50 --warmup 5 > gpurun_out/shapes/bench_$c.json 2> gpurun_out/shapes/bench_$c.err
  python -c "
import json;d=json.loads(open('gpurun_out/shapes/bench_$c.json').read().strip().splitlines()[-1]);print('$c', round(d['ms_per_step'],3), round(d['value']), d['roofline']['kernel'], round(d['roofline']['frac'],3),  d['roofline']['peak_kind'], round(d['step_roofline']['frac'],3), d['clocks']['sm_mhz'], d['cpu_baseline']['value'])"
done
timeout 800 python bench.py --steps 50 --warmup 5 > gpurun_out/shapes/bench_cfg4.json 2> gpurun_out/shapes/bench_cfg4.err
python -c "
import json;d=json.loads(open('gpurun_out/shapes/bench_cfg4.json').read().strip().splitlines()[-1]);print('cfg4', round(d['ms_per_step'],3), round(d['value']), d['roofline']['kernel'], round(d['roofline']['frac'],3), d['roofline']['peak_kind'], round(d['step_roofline']['frac'],3), d['clocks']['sm_mhz'], d['cpu_baseline']['value'])"
