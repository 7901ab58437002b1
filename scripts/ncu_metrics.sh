#!/bin/bash
# Few-metric ncu pass of one kernel under several env settings:
#   bash scripts/ncu_metrics.sh <cfg> <kernel-regex> "ENV=a" "ENV=b" ...
CFG=$1; KRE=$2; shift 2
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex.sum
for envs in "$@"; do
  env $envs timeout 600 /usr/local/cuda/bin/ncu --metrics $M --clock-control none -k regex:"$KRE" -c 1 --csv \
     python bench.py --config $CFG --profile-steps 1 2>/dev/null | python3 -c '
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
hdr=rows[0]; mi=hdr.index("Metric Name"); vi=hdr.index("Metric Value"); ui=hdr.index("Metric Unit")
print(" ".join("%s=%s%s"%(r[mi].split("__")[1][:28],r[vi],r[ui]) for r in rows[1:]))
' | sed "s/^/[$envs] /"
done
