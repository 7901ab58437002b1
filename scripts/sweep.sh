#!/bin/bash
# Quick A/B of kernel variants via env vars: bash scripts/sweep.sh <cfg> "ENV1=a ENV2=b" "ENV1=c" ...
CFG=$1; shift
for envs in "$@"; do
  line=$(env $envs timeout 300 python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/tmp/err.txt | tail -1)
  echo "[$envs] $(echo "$line" | python3 -c '
import json,sys
try:
  d=json.loads(sys.stdin.read()); k=d["kernels"]
  print("ms/step=%.3f recon=%.3fms (%.0f TF/s) attn=%.3fms (%.0f GB/s) comb=%.3f frac_step=%.3f clk=%s" % (d["ms_per_step"], (k.get("recon_gemm") or k.get("fused_step"))["ms"], (k.get("recon_gemm") or k.get("fused_step"))["achieved"] or 0, k["attention"]["ms"], k["attention"]["achieved"] or 0, k["combine"]["ms"], d["step_roofline"]["frac"], d["clocks"]))
except Exception as e: print("ERR", e)
')"
  tail -3 /tmp/err.txt
done
