# per-kernel launch list of the absorbed path on cfg4 (ncu, cold/serialised)
mkdir -p gpurun_out
timeout 600 ncu --kernel-name regex:"qt_tc|score_tc|rescale_kernel|z_tc|wv_tc|attn_pipe|combine" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
  --clock-control none --csv --log-file gpurun_out/absorb_launches.csv python bench.py --absorb --profile-steps 2 --warmup 1 ${ABS_ARGS} > gpurun_out/absorb_ncu.log 2>&1
tail -3 gpurun_out/absorb_ncu.log
