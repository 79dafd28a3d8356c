#!/bin/bash
# ncu evidence for the final kernels (register floors): C3 iteration pair (--set full), C4 rank
# kernels (time + DRAM bytes), launch list of the first ~12000 launches of the default bench command.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:EpiXIter|EpiYIter' -s 20 -c 2 -o gpurun_out/r02_c3_fin_iter python scripts/prof_iter.py --config c3 --reps 1 --steps 20 > gpurun_out/ncu_fin_c3.log 2>&1
python scripts/ncu_summary.py gpurun_out/r02_c3_fin_iter.ncu-rep > gpurun_out/r02_c3_fin_iter_summary.txt 2>&1
timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --kernel-name-base demangled \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --csv --log-file gpurun_out/r02_c4_fin_kernels.csv python scripts/prof_c4.py --reps 1 --profile > gpurun_out/c4_fin_ncu.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/r02_c3_fin_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_fin_ncu.log 2>&1
echo done > gpurun_out/ncu_fin_done.txt
