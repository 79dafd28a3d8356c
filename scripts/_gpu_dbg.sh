#!/bin/bash
mkdir -p gpurun_out
for v in epa3; do
HPR_LIB_PATH=$PWD/paper_2408_12179_b200/variants/libhprlp_b200_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -k "many_blocks" -x -q -rf > gpurun_out/pytest_dbg_$v.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dbg_$v.log
done
