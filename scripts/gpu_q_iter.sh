# quantile-mode iteration: exactness tests, then the headline bench
timeout 900 python -m pytest tests/test_gpu_quantiles.py tests/test_gpu_point_parity.py tests/test_gpu_generated.py -x -q -p no:cacheprovider > gpurun_out/r02_q_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02_q_tests.log
tail -3 gpurun_out/r02_q_tests.log
timeout 900 python bench.py --no-cpu-baseline --no-trace --no-c5 > gpurun_out/r02_q_bench.log 2>&1; echo "bench exit $?"
tail -c 1500 gpurun_out/r02_q_bench.log
