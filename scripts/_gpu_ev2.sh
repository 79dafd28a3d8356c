#!/bin/bash
# Final-kernel captures: ncu --set full of the C3 iteration pair, launch list of one C3 bench step.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:EpiXIter|EpiYIter' -s 20 -c 2 -o gpurun_out/r02_c3_final_iter python scripts/prof_iter.py --config c3 --reps 1 --steps 20 > gpurun_out/ncu_full_c3.log 2>&1
python scripts/ncu_summary.py gpurun_out/r02_c3_final_iter.ncu-rep > gpurun_out/r02_c3_final_iter_summary.txt 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c3_bench_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_ncu.log 2>&1
