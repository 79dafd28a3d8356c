#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/variants2.log; : > $out
for cfg in c2 c3; do
  for so in paper_2408_12179_b200/variants/*.so; do
    echo "== $cfg $(basename $so)" >> $out
    HPR_LIB_PATH=$PWD/$so timeout 600 python scripts/prof_iter.py --config $cfg --reps 3 2>&1 | grep per-it >> $out
  done
done
# steady-state per-kernel durations (no cache flush) of the iteration kernels
for cfg in c2 c3; do
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --kernel-name-base demangled -k 'regex:EpiXIter|EpiYIter' -s 40 -c 6 --csv --log-file gpurun_out/steady_$cfg.csv python scripts/prof_iter.py --config $cfg --reps 1 --steps 30 > /dev/null 2>&1
done
