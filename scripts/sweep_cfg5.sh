#!/bin/bash
# cfg5 hidden-fraction sweep (OPT-66B contexts, 1 GPU).  Short steps get more of them so the
# timed region outlasts nvidia-smi's 100 ms sampling (clocks measured under load).
OUT=gpurun_out/${SWEEP_TAG:-sweep}; mkdir -p $OUT
for h in ${H_LIST:-0.0 0.015625 0.03125 0.0625 0.125 0.25 0.5 0.75 1.0}; do
  steps=$(python -c "print(300 if $h <= 0.0625 else (60 if $h <= 0.25 else 20))")
  timeout 600 python bench.py --config cfg5:$h --steps $steps --warmup 3 --no-cpu-baseline --no-e2e $SWEEP_ARGS > $OUT/cfg5_$h.json 2>/dev/null
  python3 -c "
import json; d=json.load(open('$OUT/cfg5_$h.json')); k=d['kernels']
g=(k.get('recon_gemm') or k.get('fused_step') or k.get('absorbed_hidden') or {'ms': 0.0})
c=d['clocks'] or {}
print('h=$h', 'steps=$steps', 'ms=%.3f'%d['ms_per_step'], 'req/s=%.0f'%d['value'], 'gemm=%.3f'%g['ms'], 'Troof=%.3f'%d['step_roofline']['T_roof_ms'], 'frac=%.3f'%d['step_roofline']['frac'], c.get('sm_mhz'), c.get('power_w'), c.get('reasons'))"
done
