#!/bin/bash
OUT=gpurun_out/sweep; mkdir -p $OUT
for h in ${H_LIST:-0.0 0.015625 0.03125 0.0625 0.125 0.25 0.5 0.75 1.0}; do
  timeout 600 python bench.py --config cfg5:$h --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/cfg5_$h.json 2>/dev/null
  python3 -c "
import json; d=json.load(open('$OUT/cfg5_$h.json')); k=d['kernels']
print('h=$h', 'ms=%.3f'%d['ms_per_step'], 'req/s=%.0f'%d['value'], 'recon=%.3f'%(k.get('recon_gemm') or k.get('fused_step'))['ms'], 'attn=%.3f'%k['attention']['ms'], 'Troof=%.3f'%d['step_roofline']['T_roof_ms'], 'frac=%.3f'%d['step_roofline']['frac'], d['clocks']['sm_mhz'])"
done
