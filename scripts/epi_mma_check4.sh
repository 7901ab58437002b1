cd $GRAFT_REPO_ROOT
python -c "from paper_2504_07494_b200 import build as b; b.build()"
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 | tee gpurun_out/full_pytest.txt
HC_EPI_MMA=2 timeout 600 python -m pytest tests -m gpu -q -k "rope" 2>&1 | tail -4 | tee -a gpurun_out/full_pytest.txt
TAG=epi_mma4 REPS=2 STEPS=50 CFGS='llama3-8b' VARIANTS='base|HC_EPI_MMA=0' bash scripts/ab_run.sh
for c in llama3-8b yi-6b; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2>/dev/null; done
timeout 600 python bench.py --config llama3-8b --rope 500000 --no-cpu-baseline > gpurun_out/bench_llama3-8b_rope.json 2>/dev/null
timeout 600 python bench.py --config llama3-8b --rope 500000 --no-cpu-baseline > gpurun_out/bench_llama3-8b_rope.json 2>/dev/null
HC_EPI_MMA=0 timeout 600 python bench.py --config llama3-8b --rope 500000 --no-cpu-baseline --steps 20 > gpurun_out/bench_llama3-8b_rope_rowepi.json 2>/dev/null
for f in gpurun_out/bench_*.json; do python3 -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), d['clocks']['sm_mhz'])"; done
