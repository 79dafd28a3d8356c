#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_batch_solve -c 1 -o gpurun_out/prof_batch python scripts/batch_time.py 148 > gpurun_out/ncu_batch.log 2>&1
