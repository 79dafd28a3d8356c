mkdir -p gpurun_out
CS="compute-sanitizer --target-processes all --print-limit 50 --error-exitcode 7"
timeout 600 $CS --tool initcheck python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/sanitize_smoke_initcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_smoke_initcheck.log
timeout 1200 $CS --tool racecheck python -m pytest -v tests/test_gpu_parity.py -k "test_iteration_bit_exact_c1 or test_scaling_and_power or test_spmv_abi or test_edge_shapes_bit_exact" > gpurun_out/sanitize_engines_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_engines_racecheck.log
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c1 --steps 20 --warmup 3 > gpurun_out/bench_c1.log 2>&1
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2>&1
bash scripts/r02_variants.sh
