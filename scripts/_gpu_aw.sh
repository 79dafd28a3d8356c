#!/bin/bash
# TS index words (HPR_TS_AW): parity tests, then C3 per-iteration A/B against the
# pre-change library (variants/libhprlp_b200_head.so), alternating, same box.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "ts or flow" > gpurun_out/aw_tests.log 2>&1; echo "rc=$?" >> gpurun_out/aw_tests.log
out=gpurun_out/aw_ab.log; : > $out
for rep in 1 2; do
  echo "== head" >> $out; HPR_LIB_PATH=$PWD/paper_2408_12179_b200/variants/libhprlp_b200_head.so timeout 600 python scripts/prof_iter.py --config c3 --reps 3 >> $out 2>&1
  echo "== aw1" >> $out; HPR_TS_AW=1 timeout 600 python scripts/prof_iter.py --config c3 --reps 3 >> $out 2>&1
  echo "== aw0" >> $out; HPR_TS_AW=0 timeout 600 python scripts/prof_iter.py --config c3 --reps 3 >> $out 2>&1
done
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
