#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 600 python scripts/e2e_profile.py > gpurun_out/e2e_profile.log 2>&1
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2>&1
timeout 900 python bench.py --config c4 --c4-rows 200000 --steps 2 --warmup 3 > gpurun_out/bench_c4_small.log 2>&1
timeout 900 python bench.py --impl reference --config c5 --steps 1 --warmup 3 > gpurun_out/bench_ref_c5.log 2>&1
