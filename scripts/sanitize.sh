#!/bin/bash
OUT=gpurun_out/san; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --print-limit 20 python scripts/sanitize_run.py > $OUT/$tool.txt 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|err|done|Error" $OUT/$tool.txt | tail -12
done
