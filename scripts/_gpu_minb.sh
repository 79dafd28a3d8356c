#!/bin/bash
# SELL register cap (HPR_SELL_MINB 6 default / 7 / 8) for the non-gather-ahead instances
# (C3's y-phase), alternating, same box: C3 and C2 per-iteration time.
mkdir -p gpurun_out
out=gpurun_out/minb_ab.log; : > $out
V=paper_2408_12179_b200/variants
for rep in 1 2; do
  for cfg in c3 c2; do
    echo "== $cfg default" >> $out; timeout 600 python scripts/prof_iter.py --config $cfg --reps 3 2>&1 | grep per-iter >> $out
    for v in minb7 minb8; do
      echo "== $cfg $v" >> $out; HPR_LIB_PATH=$PWD/$V/libhprlp_b200_$v.so timeout 600 python scripts/prof_iter.py --config $cfg --reps 3 2>&1 | grep per-iter >> $out
    done
  done
done
