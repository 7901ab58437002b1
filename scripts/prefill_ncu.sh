# per-kernel launch list of the prefill layer (OPT-66B, 8 x L) for both attention kernels
mkdir -p gpurun_out
for tc in 1 0; do
HC_PREFILL_TC=$tc timeout 600 ncu --kernel-name regex:"prefill|dense|pair|tc2" --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active \
  --clock-control none --csv --log-file gpurun_out/prefill_launches_tc$tc.csv python bench.py --mode prefill --prefill-len ${L:-2048} --prefill-reqs 8 --profile-steps 1 --warmup 1 > /dev/null 2>&1
done
