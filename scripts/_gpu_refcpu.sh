#!/bin/bash
# bench lines with the reference's own iteration as cpu_baseline (same run, same instance)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3_refcpu.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3_refcpu.log
timeout 600 python bench.py --config c2 --steps 20 --warmup 3 > gpurun_out/bench_c2_refcpu.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c2_refcpu.log
timeout 600 python bench.py --config c1 --steps 20 --warmup 3 > gpurun_out/bench_c1_refcpu.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c1_refcpu.log
