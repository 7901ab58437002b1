#!/bin/bash
# Round profile set (run under gpurun): bench lines (cfg4 with the cpu baseline; cfg2, cfg3,
# the GQA layers), the cfg4 launch list, and ncu --set full of the fused step kernel at cfg4,
# at the crossover (cfg5 1/32) and on LLaMA-3-8B (GQA), plus the KV-only attention kernel.
TAG=${1:-r02}; OUT=gpurun_out/$TAG; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
REP=/tmp/ncu_$TAG; mkdir -p $REP   # full reports stay on the box (gpurun copies back <= 64 MiB); CSV exports come back
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
timeout 900 python bench.py > $OUT/bench_cfg4.json 2> $OUT/bench_cfg4.err
for c in cfg2 cfg3 llama3-8b yi-6b; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2>/dev/null
done
timeout 600 python bench.py --config cfg4 --absorb --no-cpu-baseline > $OUT/bench_cfg4_absorb.json 2>/dev/null
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:"recon|attn|combine|fused|append" \
   --csv --log-file $OUT/launches_cfg4.csv python bench.py --profile-steps 3 > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"fused_step" -c 1 \
   -o $REP/full_fused_cfg4 python bench.py --profile-steps 1 > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"fused_step" -c 1 \
   -o $REP/full_fused_cfg5_h1_32 python bench.py --config cfg5:1/32 --profile-steps 1 > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"fused_step" -c 1 \
   -o $REP/full_fused_llama3 python bench.py --config llama3-8b --profile-steps 1 > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"attn_pipe" -c 1 \
   -o $REP/full_attn_cfg5h0 python bench.py --config cfg5:0 --profile-steps 1 > /dev/null 2>&1
for r in $REP/*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  $NCU -i $r --page details --csv > $OUT/$b.details.csv 2>/dev/null
  $NCU -i $r --page raw --csv > $OUT/$b.raw.csv 2>/dev/null
done
ls -la $OUT
