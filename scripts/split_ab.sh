# gpurun: bench A/B of the KV split size (pool split_tokens) at the given configs
cd $GRAFT_REPO_ROOT
for CFG in $CFGS; do for i in 1 2; do for S in ${SPLITS:-0 1024 2048}; do
  timeout 600 python bench.py --config $CFG --split-tokens $S --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-graph 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$CFG split=$S', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), d['clocks']['sm_mhz'])" | tee -a gpurun_out/split_ab.txt
done; done; done
