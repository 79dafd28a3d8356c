mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu --format=csv > gpurun_out/nvsmi_d.txt
timeout 1500 python -m pytest tests -m gpu -x -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
out=gpurun_out/r02_variants3.log; : > $out
for rep in 1 2; do
  for so in paper_2408_12179_b200/variants/*.so; do
    echo "== c3 $(basename $so)" >> $out
    HPR_LIB_PATH=$PWD/$so timeout 600 python scripts/prof_iter.py --config c3 --reps 3 >> $out 2>&1
  done
done
for c in c1 c2; do timeout 300 python scripts/c1_breakdown.py $c > gpurun_out/breakdown_$c.log 2>&1; done
HPR_SMALL=0 timeout 300 python scripts/c1_breakdown.py c1 > gpurun_out/breakdown_c1_graph.log 2>&1
timeout 600 python scripts/c5_pipe_sweep.py > gpurun_out/c5_pipe_sweep.log 2>&1
timeout 600 python bench.py --config c1 --steps 20 --warmup 3 > gpurun_out/bench_c1.log 2>&1
