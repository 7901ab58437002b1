# timeline variants for gpurun: VARIANTS ('|'-separated env sets), CFGS
cd $GRAFT_REPO_ROOT
python -c "from paper_2504_07494_b200 import build as b; b.build(variant='diag')"
IFS='|' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  ENVS=""; [ "$v" != "base" ] && ENVS="$v"
  echo "[$v]" | tee -a gpurun_out/${TAG:-tl}.txt
  env $ENVS REPS=10 timeout 300 python scripts/timeline.py $CFGS 2>&1 | tail -3 | tee -a gpurun_out/${TAG:-tl}.txt
done
