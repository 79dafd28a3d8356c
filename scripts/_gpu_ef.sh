#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/ef_ab.log; : > $out
for rep in 1 2; do
for so in paper_2408_12179_b200/libhprlp_b200.so paper_2408_12179_b200/variants/*.so; do
  echo "== $(basename $so)" >> $out
  HPR_LIB_PATH=$PWD/$so timeout 150 python scripts/prof_iter.py --config c3 --reps 3 2>&1 | grep per-iter >> $out
done
done
timeout 400 ncu --replay-mode application --cache-control none --clock-control none --kernel-name-base demangled \
  -k regex:"EpiXIter|EpiYIter" --launch-skip 10 --launch-count 2 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  python scripts/prof_iter.py --config c3 --steps 4 --reps 1 > gpurun_out/ncu_ss_ef.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_scale.py -m gpu -x -q > gpurun_out/pytest_ef.log 2>&1; echo rc=$? >> gpurun_out/pytest_ef.log
