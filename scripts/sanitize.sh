#!/bin/bash
OUT=gpurun_out/san; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tmem_slot_race scripts/tmem_slot_race.cu
timeout 300 $CS --tool racecheck /tmp/tmem_slot_race > $OUT/tmem_slot_race.txt 2>&1
echo "== tmem slot reproducer"; grep -E "variant|RACECHECK SUMMARY|Race reported" $OUT/tmem_slot_race.txt | sort | uniq -c | head
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --print-limit 20 python scripts/sanitize_run.py > $OUT/$tool.txt 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|err|done|Error" $OUT/$tool.txt | tail -12
done
