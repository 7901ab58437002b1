# gpurun: DRAM bytes of one fused-kernel launch (ncu, a few metrics) + bench time per variant
cd $GRAFT_REPO_ROOT
python -c "from paper_2504_07494_b200 import build as b; b.build()"
NCU=/usr/local/cuda/bin/ncu; OUT=gpurun_out/${TAG:-traffic}; mkdir -p $OUT
IFS='|' read -ra VS <<< "$VARIANTS"
for CFG in $CFGS; do
for v in "${VS[@]}"; do
  ENVS=""; [ "$v" != "base" ] && ENVS="$v"
  env $ENVS timeout 600 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum \
      --clock-control none -k regex:fused_step -c 1 --csv python bench.py --config $CFG --profile-steps 1 2>/dev/null \
      | grep -E "dram__|gpu__time|tensor|lts__t_bytes" | awk -F'","' -v v="$v" -v c="$CFG" '{print c, "["v"]", $(NF-2), $(NF-1), $NF}' | tr -d '"' | tee -a $OUT/ncu.txt
done; done
[ -n "$AB" ] && VARIANTS="$VARIANTS" bash scripts/ab_run.sh
true
