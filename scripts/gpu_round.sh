#!/bin/bash
# One GPU session: tests, bench, ncu launch list + full capture of the two hot kernels.
# Usage (under gpurun): bash scripts/gpu_round.sh <tag> [tests|notests] [config]
TAG=${1:-r1}; TESTS=${2:-tests}; CFG=${3:-cfg4}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
if [ "$TESTS" = "tests" ]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
  timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1
  tail -5 $OUT/pytest_gpu.txt
fi
timeout 600 python bench.py --config $CFG > $OUT/bench.json 2> $OUT/bench.err; tail -c 3000 $OUT/bench.json
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:"recon|attn|combine|append" \
   --csv --log-file $OUT/launches.csv python bench.py --config $CFG --profile-steps 3 > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"recon_tc|attn_pipe" -c 2 \
   -o $OUT/prof python bench.py --config $CFG --profile-steps 1 > $OUT/ncu_full.log 2>&1
ls -la $OUT
