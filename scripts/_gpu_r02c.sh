mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
out=gpurun_out/r02_variants2.log; : > $out
for rep in 1 2; do
  for cfg in c3 c2; do
    for so in paper_2408_12179_b200/variants/*.so; do
      echo "== $cfg $(basename $so)" >> $out
      HPR_LIB_PATH=$PWD/$so timeout 600 python scripts/prof_iter.py --config $cfg --reps 3 >> $out 2>&1
    done
  done
done
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3.log 2>&1
