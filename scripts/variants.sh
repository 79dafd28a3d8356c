#!/bin/bash
# time the per-iteration pair for each unroll variant on each config
for cfg in c2 c3-lite c3; do
  for u in 2 4 8; do
    echo "== u=$u"; HPR_LIB_PATH=$PWD/paper_2408_12179_b200/libhprlp_b200_u$u.so timeout 600 python scripts/prof_iter.py --config $cfg --reps 3 2>&1 | tail -2
  done
done
