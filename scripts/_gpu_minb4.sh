#!/bin/bash
# final register floors (7 reduction-free, 8 for the A_g^T partial store, 7 for the
# column-split carry blocks) vs the library before the floors changed (head6):
# GPU suite, C4 / C2 per-iteration A/B, C4 bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_minb4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_minb4.log
out=gpurun_out/minb4_ab.log; : > $out
H=$PWD/paper_2408_12179_b200/variants/libhprlp_b200_head6.so
for rep in 1 2; do
  echo "== c4 head6" >> $out; HPR_LIB_PATH=$H timeout 600 python scripts/prof_c4.py --reps 3 2>&1 | grep per-iter >> $out
  echo "== c4 final" >> $out; timeout 600 python scripts/prof_c4.py --reps 3 2>&1 | grep per-iter >> $out
  echo "== c2 head6" >> $out; HPR_LIB_PATH=$H timeout 600 python scripts/prof_iter.py --config c2 --reps 3 2>&1 | grep per-iter >> $out
  echo "== c2 final" >> $out; timeout 600 python scripts/prof_iter.py --config c2 --reps 3 2>&1 | grep per-iter >> $out
done
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 > gpurun_out/bench_c4_minb4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4_minb4.log
