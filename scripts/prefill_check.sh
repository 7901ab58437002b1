# f3 prefill: parity for every tcgen05 configuration, then the OPT-66B prefill A/B (8 x 2048, 8 x 4096)
mkdir -p gpurun_out
for cfg in 2 1 128; do
  HC_PREFILL_CFG=$cfg timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill" --timeout 600 2>&1 | tail -1
done
for cfg in 2 1; do
  for L in 2048 4096; do
    HC_PREFILL_CFG=$cfg timeout 600 python bench.py --mode prefill --prefill-len $L --prefill-reqs 8 --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('cfg=$cfg L=$L', round(d['ms_per_step'],3), round(d['value']))"
  done
  HC_PREFILL_CFG=$cfg timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:"prefill_attn_tc" --clock-control none --csv --log-file gpurun_out/pf_$cfg.csv python bench.py --mode prefill --prefill-len 2048 --prefill-reqs 8 --profile-steps 1 --warmup 1 > /dev/null 2>&1
  grep prefill_attn gpurun_out/pf_$cfg.csv | awk -F'","' '{print "cfg='$cfg'", $(NF-2), $NF}' | head -2
done
