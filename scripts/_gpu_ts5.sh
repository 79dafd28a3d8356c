#!/bin/bash
# TS default (x-phase of C3) : GPU suite, x-phase variant sweep, C3 bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
out=gpurun_out/ts_var.log; : > $out
for rep in 1 2; do
for so in paper_2408_12179_b200/libhprlp_b200.so paper_2408_12179_b200/variants/*.so; do
  echo "== $(basename $so)" >> $out
  HPR_LIB_PATH=$PWD/$so timeout 120 python scripts/prof_iter.py --config c3 --reps 3 2>&1 | grep -E "per-iter|layout" >> $out
done
done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
