# f4 (ii) absorbed path: cfg4 bench line, cfg5 hidden-fraction sweep, launch list, ncu --set full of z_tc
OUT=gpurun_out/absorb; mkdir -p $OUT
timeout 300 python bench.py --absorb --steps 50 --warmup 5 --no-cpu-baseline > $OUT/bench_cfg4.json 2>$OUT/bench_cfg4.err
for h in 0.0 0.03125 0.125 0.5 1.0; do
  timeout 600 python bench.py --absorb --config cfg5:$h --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/cfg5_$h.json 2>/dev/null
  python3 -c "
import json; d=json.load(open('$OUT/cfg5_$h.json')); k=d['kernels']
print('h=$h', 'ms=%.3f'%d['ms_per_step'], 'req/s=%.0f'%d['value'], 'hidden=%.3f'%(k.get('absorbed_hidden') or {'ms':0})['ms'], 'attn=%.3f'%k['attention']['ms'], 'Troof=%.3f'%d['step_roofline']['T_roof_ms'], 'frac=%.3f'%d['step_roofline']['frac'], d['clocks']['sm_mhz'])"
done
timeout 600 ncu --kernel-name regex:"qt_kernel|score_tc|rescale_kernel|z_tc|wv_kernel|attn_pipe|combine" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches_cfg4.csv python bench.py --absorb --profile-steps 2 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --kernel-name regex:"z_tc|score_tc" --launch-count 2 --set full --clock-control none --import-source on \
  -o $OUT/absorb_full python bench.py --absorb --profile-steps 1 --warmup 0 > $OUT/ncu_full.log 2>&1
ncu -i $OUT/absorb_full.ncu-rep --page details --csv > $OUT/absorb_full_details.csv 2>/dev/null
ls -la $OUT
