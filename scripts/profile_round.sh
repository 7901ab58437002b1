#!/bin/bash
# Round profile set: launch list (cfg4), ncu --set full of the GEMM (cfg4) and of the
# attention kernel (cfg5 h=0, KV-only, where it dominates), plus the default bench line.
TAG=${1:-r01}; OUT=gpurun_out/$TAG; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 900 python bench.py > $OUT/bench_cfg4.json 2> $OUT/bench_cfg4.err
timeout 600 python bench.py --config cfg5:0.0 --no-cpu-baseline > $OUT/bench_cfg5_h0.json 2>/dev/null
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:"recon|attn|combine|fused" \
   --csv --log-file $OUT/launches_cfg4.csv python bench.py --profile-steps 3 > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"fused_step" -c 1 \
   -o $OUT/full_fused_cfg4 python bench.py --profile-steps 1 > /dev/null 2>&1
HC_FUSED=0 timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"recon_tc2" -c 1 \
   -o $OUT/full_recon_cfg4 python bench.py --profile-steps 1 > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"attn_pipe" -c 1 \
   -o $OUT/full_attn_cfg5h0 python bench.py --config cfg5:0.0 --profile-steps 1 > /dev/null 2>&1
ls -la $OUT
for r in full_fused_cfg4 full_recon_cfg4 full_attn_cfg5h0; do
  [ -f $OUT/$r.ncu-rep ] && $NCU -i $OUT/$r.ncu-rep --page details --csv > $OUT/$r.csv 2>/dev/null
done
ls -la $OUT
