#!/bin/bash
# One GPU session: tests, smoke, per-iteration timing, bench line, ncu launch list.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for c in c2 c3; do timeout 600 python scripts/prof_iter.py --config $c --reps 3 > gpurun_out/prof_$c.log 2>&1; done
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:EpiXIter|EpiYIter' -s 4 -c 2 -o gpurun_out/prof_c3_iter python scripts/prof_iter.py --config c3 --reps 1 --steps 10 > gpurun_out/ncu_full.log 2>&1
cuobjdump -sass paper_2408_12179_b200/libhprlp_b200.so > gpurun_out/sass.txt 2>&1
