cd $GRAFT_REPO_ROOT
python -c "from paper_2504_07494_b200 import build as b; b.build()"
HC_EPI_MMA=2 timeout 900 python -m pytest tests -m gpu -x -q -k "gqa or mixed_batch or opt_shaped or all_heads or high_dynamic or boundary or decode_layer or attend_epilogue or fused" 2>&1 | tail -8 | tee gpurun_out/epi_mma_pytest.txt
TAG=epi_mma REPS=2 STEPS=50 CFGS='llama3-8b yi-6b cfg4 cfg2' VARIANTS='base|HC_EPI_MMA=2|HC_LIB_FILE=libhc_head.so' bash scripts/ab_run.sh
