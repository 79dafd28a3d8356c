mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_exact.py tests/test_gpu_config_scale.py -q -m gpu -k "exact or c3_trajectory" -rf > gpurun_out/exact_tests.log 2>&1; echo "rc=$?" >> gpurun_out/exact_tests.log
timeout 300 python scripts/exact_time.py > gpurun_out/exact_time.log 2>&1
