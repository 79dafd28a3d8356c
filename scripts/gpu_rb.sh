#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rowblock.py -x -q > gpurun_out/pytest_rb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rb.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:EpiXIter|EpiYIter' -s 4 -c 2 -o gpurun_out/prof_c2_iter python scripts/prof_iter.py --config c2 --reps 1 --steps 10 > gpurun_out/ncu_full_c2.log 2>&1
