#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "bit_exact" > gpurun_out/pytest_cb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cb.log
out=gpurun_out/cb2.log; : > $out
for cb in 0 1; do
  echo "== c2 HPR_CB=$cb" >> $out
  HPR_CB=$cb timeout 600 python scripts/prof_iter.py --config c2 --reps 3 >> $out 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active --cache-control none --clock-control none --kernel-name-base demangled -k 'regex:k_cb' -s 20 -c 4 --csv --log-file gpurun_out/cb2_steady.csv env HPR_CB=1 python scripts/prof_iter.py --config c2 --reps 1 --steps 20 > /dev/null 2>&1
