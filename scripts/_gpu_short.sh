#!/bin/bash
# TS compact single-batch path (HPR_TS_SHORT): TS parity tests, then C3 per-iteration
# A/B against the library before it (variants/libhprlp_b200_head.so), alternating.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "ts or flow or c3 or rowblock" > gpurun_out/short_tests.log 2>&1; echo "rc=$?" >> gpurun_out/short_tests.log
out=gpurun_out/short_ab.log; : > $out
V=paper_2408_12179_b200/variants
for rep in 1 2; do
  echo "== head" >> $out; HPR_LIB_PATH=$PWD/$V/libhprlp_b200_head.so timeout 600 python scripts/prof_iter.py --config c3 --reps 3 >> $out 2>&1
  echo "== short" >> $out; timeout 600 python scripts/prof_iter.py --config c3 --reps 3 >> $out 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:EpiXIter' -s 10 -c 1 -o gpurun_out/r02_c3_short_x python scripts/prof_iter.py --config c3 --reps 1 --steps 20 > gpurun_out/ncu_short.log 2>&1
python scripts/ncu_summary.py gpurun_out/r02_c3_short_x.ncu-rep > gpurun_out/r02_c3_short_x_summary.txt 2>&1
