# gpurun: ncu --set full with source-level stall sampling of the fused kernel at one config;
# exports the source page (SASS + per-instruction stall samples) as CSV
cd $GRAFT_REPO_ROOT
CFG=${CFG:-cfg5:1/32}; TAG=${TAG:-src}; OUT=gpurun_out/$TAG; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"${KERNEL:-fused_step}" -c 1 \
   -o /tmp/$TAG python bench.py --config $CFG --profile-steps 1 > $OUT/ncu.log 2>&1
$NCU -i /tmp/$TAG.ncu-rep --page source --csv --print-source sass > $OUT/source_sass.csv 2>$OUT/src.err
$NCU -i /tmp/$TAG.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
$NCU -i /tmp/$TAG.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
ls -la $OUT; tail -3 $OUT/ncu.log
