#!/bin/bash
# Generic same-box A/B of library knobs (internal.h Tuning; read at pool create).
#   VARIANTS="base|HC_L2HINT=3|HC_LIB_FILE=libhc_base.so" STEPS=100 bash scripts/env_ab.sh cfg5:1/32 cfg4
# Each variant runs REPS times, interleaved, so box state (power, clocks) drifts evenly.
VARIANTS=${VARIANTS:-base}
IFS='|' read -ra VS <<< "$VARIANTS"
for CFG in "$@"; do
for i in $(seq ${REPS:-2}); do
for v in "${VS[@]}"; do
  ENVS=""; [ "$v" != "base" ] && ENVS="$v"
  env $ENVS timeout 600 python bench.py --config $CFG --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline --no-e2e --no-graph \
    2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d.get('clocks') or {}; p=d['step_ms_percentiles']
print('$CFG', '[$v]', 'ms', round(d['ms_per_step'],3), 'p50', round(p['p50'],3), 'frac', round(d['step_roofline']['frac'],3), 'MHz', c.get('sm_mhz'), 'W', c.get('power_w'))"
done; done; done
