#!/bin/bash
# C2: both x-phase engines (staged, SELL) against the oracle's C kernels over 40 fused iterations.
# (A compute-sanitizer pass over the TS index-word kernel was attempted in the same call; the
# pool has since closed compute-sanitizer, so the earlier r02_sanitize_* logs are the last ones.)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "c2_engines" > gpurun_out/c2_engines.log 2>&1; echo "rc=$?" >> gpurun_out/c2_engines.log
