# gpurun: end-of-round profile set (profile_round.sh) + cfg5 sweep
cd $GRAFT_REPO_ROOT
python -c "from paper_2504_07494_b200 import build as b; b.build()"
bash scripts/profile_round.sh ${TAG:-r02}
SWEEP_TAG=${TAG:-r02}_sweep bash scripts/sweep_cfg5.sh 2>&1 | tee gpurun_out/${TAG:-r02}_sweep.txt
