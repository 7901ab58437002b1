cd $GRAFT_REPO_ROOT
python -c "from paper_2504_07494_b200 import build as b; b.build()"
timeout 900 python -m pytest tests -m gpu -q -k "mma or gqa" 2>&1 | tail -15 | tee gpurun_out/epi_mma3_pytest.txt
HC_EPI_MMA=2 timeout 900 python -m pytest tests -m gpu -q -k "high_dynamic or all_heads or mixed_batch" 2>&1 | tail -15 | tee -a gpurun_out/epi_mma3_pytest.txt
TAG=epi_mma3 REPS=2 STEPS=50 CFGS='llama3-8b yi-6b' VARIANTS='base|HC_EPI_MMA=0|HC_LIB_FILE=libhc_head.so' bash scripts/ab_run.sh
