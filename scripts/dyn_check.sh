cd $GRAFT_REPO_ROOT
python -c "from paper_2504_07494_b200 import build as b; b.build()"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 | tee gpurun_out/dyn_pytest.txt
TAG=dyn_traffic CFGS='cfg4 cfg5:1/32' VARIANTS='base|HC_DYN_TILES=0|HC_GROUP_N=6|HC_GROUP_N=8' bash scripts/traffic_sweep.sh
TAG=dyn_ab REPS=2 STEPS=50 CFGS='cfg4 cfg5:0.03125 cfg5:0.015625 cfg5:0.0625 cfg2 llama3-8b' VARIANTS='base|HC_DYN_TILES=0' bash scripts/ab_run.sh
