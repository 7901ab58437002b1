# ncu --set full of the tcgen05 prefill attention kernel (OPT-66B, 8 x 2048) + bench lines
OUT=gpurun_out/prefill; mkdir -p $OUT
for L in 512 2048 4096; do
  timeout 600 python bench.py --mode prefill --prefill-len $L --prefill-reqs 8 --steps 10 --warmup 3 > $OUT/bench_prefill_$L.json 2>/dev/null
done
timeout 900 ncu --kernel-name regex:"prefill_attn_tc" --launch-count 1 --set full --clock-control none --import-source on \
  -o $OUT/prefill_full python bench.py --mode prefill --prefill-len 2048 --prefill-reqs 8 --profile-steps 1 --warmup 0 > $OUT/ncu.log 2>&1
ncu -i $OUT/prefill_full.ncu-rep --page details --csv > $OUT/prefill_full_details.csv 2>/dev/null
ls $OUT
