#!/bin/bash
# TS byte-ring variant: parity forced on, then C3 / C2 / C4 A/B.
mkdir -p gpurun_out
HPR_TS=1 HPR_TS_RING=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -rf > gpurun_out/pytest_tr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tr.log
out=gpurun_out/tr_ab.log; : > $out
for m in "0 2 2" "1 1 1" "1 0 1" "1 1 0"; do
  set -- $m
  echo "== c3 RING=$1 TS_A=$2 TS_AT=$3" >> $out
  HPR_TS_RING=$1 HPR_TS_A=$2 HPR_TS_AT=$3 timeout 150 python scripts/prof_iter.py --config c3 --reps 3 2>&1 | grep per-iter >> $out
done
for m in "0 0" "1 1"; do
  set -- $m
  echo "== c2 RING=$1 TS=$2" >> $out
  HPR_TS_RING=$1 HPR_TS=$2 timeout 150 python scripts/prof_iter.py --config c2 --reps 3 2>&1 | grep per-iter >> $out
  echo "== c4 RING=$1 TS=$2" >> $out
  HPR_TS_RING=$1 HPR_TS=$2 timeout 300 python scripts/prof_c4.py --reps 3 2>&1 | grep per-iter >> $out
done
