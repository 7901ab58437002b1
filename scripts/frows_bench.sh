# committed bench lines for the f-rows: decode layer (f1), RoPE (f4 i), planner timing (f2)
OUT=gpurun_out/frows; mkdir -p $OUT
timeout 900 python bench.py --mode layer --steps 20 --warmup 3 > $OUT/bench_layer_cfg4.json 2>$OUT/layer.err
timeout 900 python bench.py --rope 500000 --steps 30 --warmup 3 --no-cpu-baseline > $OUT/bench_cfg4_rope.json 2>$OUT/rope.err
python scripts/planner_timing.py > $OUT/planner_timing.json 2>$OUT/planner.err
for f in $OUT/*.json; do echo $f; head -c 400 $f; echo; done
