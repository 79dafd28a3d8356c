#!/bin/bash
# C5 (reference pool as cpu_baseline) and C4 (gather roofline) bench lines with the current bench.py
mkdir -p gpurun_out
timeout 600 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/bench_c5_v2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5_v2.log
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4_v2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4_v2.log
