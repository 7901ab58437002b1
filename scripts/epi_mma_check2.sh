cd $GRAFT_REPO_ROOT
python -c "from paper_2504_07494_b200 import build as b; b.build()"
timeout 900 python -m pytest tests -m gpu -x -q -k "gqa or rope" 2>&1 | tail -4 | tee gpurun_out/epi_mma2_pytest.txt
HC_EPI_MMA=2 timeout 900 python -m pytest tests -m gpu -x -q -k "mixed_batch or opt_shaped or all_heads or high_dynamic or boundary or decode_layer" 2>&1 | tail -4 | tee -a gpurun_out/epi_mma2_pytest.txt
TAG=epi_mma2 REPS=2 STEPS=50 CFGS='llama3-8b yi-6b' VARIANTS='base|HC_EPI_MMA=0|HC_GQA_SCRATCH=0|HC_GQA_SCRATCH=0 HC_EPI_MMA=0' bash scripts/ab_run.sh
