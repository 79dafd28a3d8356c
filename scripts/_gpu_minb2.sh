#!/bin/bash
# SELL floor of 7 resident CTAs (72 registers) for reduction-free epilogues vs the previous
# library (variants/libhprlp_b200_head6.so: 6 / 80 everywhere): GPU suite, then C3 / C4 / C2
# per-iteration A/B alternating on one box, then the default bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_minb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_minb.log
out=gpurun_out/minb2_ab.log; : > $out
H=$PWD/paper_2408_12179_b200/variants/libhprlp_b200_head6.so
for rep in 1 2; do
  for cfg in c3 c2; do
    echo "== $cfg head6" >> $out; HPR_LIB_PATH=$H timeout 600 python scripts/prof_iter.py --config $cfg --reps 3 2>&1 | grep per-iter >> $out
    echo "== $cfg minb7" >> $out; timeout 600 python scripts/prof_iter.py --config $cfg --reps 3 2>&1 | grep per-iter >> $out
  done
  echo "== c4 head6" >> $out; HPR_LIB_PATH=$H timeout 600 python scripts/prof_c4.py --reps 3 2>&1 | grep per-iter >> $out
  echo "== c4 minb7" >> $out; timeout 600 python scripts/prof_c4.py --reps 3 2>&1 | grep per-iter >> $out
done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3_minb.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3_minb.log
