#!/bin/bash
mkdir -p gpurun_out
for pf in 1 0; do
  echo "== HPR_PREFAULT=$pf" >> gpurun_out/e2e_c3.log
  HPR_PREFAULT=$pf timeout 400 python scripts/e2e_breakdown.py c3 >> gpurun_out/e2e_c3.log 2>&1
done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c3_bench_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_ncu.log 2>&1
