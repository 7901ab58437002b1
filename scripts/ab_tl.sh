# A/B (bench) then timelines for gpurun
cd $GRAFT_REPO_ROOT
bash scripts/ab_run.sh
VARIANTS="$TL_VARIANTS" TAG=${TAG}_tl bash scripts/tl_run.sh
