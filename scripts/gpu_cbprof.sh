#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,lts__t_bytes.sum,smsp__cycles_active.avg --cache-control none --clock-control none --kernel-name-base demangled -k 'regex:k_cb' -s 20 -c 4 --csv --log-file gpurun_out/cb_steady.csv python scripts/prof_iter.py --config c2 --reps 1 --steps 20 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:k_cb' -s 20 -c 2 -o gpurun_out/prof_cb python scripts/prof_iter.py --config c2 --reps 1 --steps 20 > /dev/null 2>&1
