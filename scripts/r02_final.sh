#!/bin/bash
# Round-2 closing evidence: smoke, GPU suite, bench lines for every config (+ reference
# arms at C3 / C2 / C5), ncu --set full of the C3 and C2 iteration pairs, the C4 rank's
# per-kernel DRAM traffic, launch list of one C3 bench step.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
for c in c1 c2 c5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$c.log
done
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref_c3.log
for c in c2 c5; do
  timeout 600 python bench.py --impl reference --config $c --steps 3 --warmup 3 > gpurun_out/bench_ref_$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref_$c.log
done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:EpiXIter|EpiYIter' -s 20 -c 2 -o gpurun_out/r02_c3_close_iter python scripts/prof_iter.py --config c3 --reps 1 --steps 20 > gpurun_out/ncu_full_c3.log 2>&1
python scripts/ncu_summary.py gpurun_out/r02_c3_close_iter.ncu-rep > gpurun_out/r02_c3_close_iter_summary.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:EpiXIter|EpiYIter' -s 20 -c 2 -o gpurun_out/r02_c2_close_iter python scripts/prof_iter.py --config c2 --reps 1 --steps 20 > gpurun_out/ncu_full_c2.log 2>&1
python scripts/ncu_summary.py gpurun_out/r02_c2_close_iter.ncu-rep > gpurun_out/r02_c2_close_iter_summary.txt 2>&1
timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --kernel-name-base demangled \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --csv --log-file gpurun_out/r02_c4_close_kernels.csv python scripts/prof_c4.py --reps 1 --profile > gpurun_out/c4_ncu.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c3_close_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_ncu.log 2>&1
