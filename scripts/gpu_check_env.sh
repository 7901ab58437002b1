# gpurun: GPU suite under an env setting ($TEST_ENV), then bench A/B (VARIANTS/CFGS)
cd $GRAFT_REPO_ROOT
python -c "from paper_2504_07494_b200 import build as b; b.build()"
env $TEST_ENV timeout 1200 python -m pytest tests -m gpu -x -q ${K:+-k "$K"} 2>&1 | tail -8 | tee gpurun_out/${TAG:-chk}_pytest.txt
[ -n "$VARIANTS" ] && bash scripts/ab_run.sh
true
