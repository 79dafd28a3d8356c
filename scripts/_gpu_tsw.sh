#!/bin/bash
# TS consumer warps 24 (current) / 26 / 27 (same 72-register cap: at most 7 warps per SMSP), C3, alternating.
mkdir -p gpurun_out
out=gpurun_out/tsw_ab.log; : > $out
V=$PWD/paper_2408_12179_b200/variants
for rep in 1 2; do
  for v in cur w26 w27; do
    echo "== c3 $v" >> $out; HPR_LIB_PATH=$V/libhprlp_b200_$v.so timeout 600 python scripts/prof_iter.py --config c3 --reps 3 2>&1 | grep per-iter >> $out
  done
done
