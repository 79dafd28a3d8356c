mkdir -p gpurun_out; : > gpurun_out/c5var.log
for rep in 1 2; do for so in paper_2408_12179_b200/variants/*.so; do echo "== $(basename $so)" >> gpurun_out/c5var.log; HPR_LIB_PATH=$PWD/$so timeout 600 python scripts/batch_time.py 1184 2>&1 | grep "rep 2" >> gpurun_out/c5var.log; done; done
