#!/bin/bash
# C4 rank (P=1): per-iteration with / without TS, e2e phases, kernel list of one TS replay.
mkdir -p gpurun_out
for ts in 2 0; do
  echo "== HPR_TS=$ts" >> gpurun_out/c4_ab.log
  HPR_TS=$ts timeout 300 python scripts/prof_c4.py --reps 3 >> gpurun_out/c4_ab.log 2>&1
  HPR_TS=$ts timeout 400 python scripts/c4_e2e_phases.py > gpurun_out/c4_e2e_ts$ts.log 2>&1
done
HPR_TS=2 timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --kernel-name-base demangled \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  python scripts/prof_c4.py --reps 1 --profile > gpurun_out/c4_ncu_ts.txt 2>&1
