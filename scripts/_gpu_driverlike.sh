#!/bin/bash
# the driver's own round-end commands (N=1): our arm, then the reference arm
mkdir -p gpurun_out
s=$(date +%s); timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv_ours.log 2>&1; echo "rc=$? wall=$(( $(date +%s) - s ))s" >> gpurun_out/drv_ours.log
s=$(date +%s); timeout 1800 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv_ref.log 2>&1; echo "rc=$? wall=$(( $(date +%s) - s ))s" >> gpurun_out/drv_ref.log
