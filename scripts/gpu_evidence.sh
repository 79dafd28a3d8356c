#!/bin/bash
# Round evidence: tests, smoke, bench lines (C2 headline + reference arm, C3, C4 at one GPU, C5),
# per-iteration timings, launch list of one C2 solve, ncu --set full of the iteration kernels.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_c2.log 2>&1
timeout 900 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c3.log 2>&1
timeout 1200 python bench.py --config c4 --steps 2 --warmup 3 > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 > gpurun_out/bench_c5.log 2>&1
for c in c2 c3; do timeout 600 python scripts/prof_iter.py --config $c --reps 3 > gpurun_out/prof_$c.log 2>&1; done
timeout 600 python scripts/e2e_breakdown.py > gpurun_out/e2e_breakdown.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2300 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
for c in c2 c3; do
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:EpiXIter|EpiYIter' -s 20 -c 2 -o gpurun_out/prof_${c}_iter python scripts/prof_iter.py --config $c --reps 1 --steps 20 > gpurun_out/ncu_full_$c.log 2>&1
done
