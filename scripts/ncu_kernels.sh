#!/bin/bash
# ncu --set full of the hot kernels for one config: bash scripts/ncu_kernels.sh <tag> <cfg> <kernel-regex> [count]
TAG=$1; CFG=$2; KRE=$3; CNT=${4:-1}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c $CNT \
   -o $OUT/prof_$CFG python bench.py --config $CFG --profile-steps 1 > $OUT/ncu_$CFG.log 2>&1
tail -3 $OUT/ncu_$CFG.log
