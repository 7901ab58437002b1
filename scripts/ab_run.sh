# ad-hoc A/B driver for gpurun: VARIANTS / CFGS / REPS / STEPS from the caller
cd $GRAFT_REPO_ROOT
python -c "from paper_2504_07494_b200 import build as b; b.build()"
START=$(date +%s)
VARIANTS="$VARIANTS" REPS=${REPS:-1} STEPS=${STEPS:-100} bash scripts/env_ab.sh $CFGS 2>&1 | tee -a gpurun_out/${TAG:-ab}.txt
echo elapsed $(( $(date +%s) - START ))
