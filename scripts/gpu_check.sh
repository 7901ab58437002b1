# gpurun: GPU parity tests (subset with -k via $K) then bench A/B
cd $GRAFT_REPO_ROOT
python -c "from paper_2504_07494_b200 import build as b; b.build()"
timeout 900 python -m pytest tests -m gpu -x -q ${K:+-k "$K"} 2>&1 | tail -5 | tee gpurun_out/${TAG:-chk}_pytest.txt
[ -n "$VARIANTS" ] && bash scripts/ab_run.sh
true
