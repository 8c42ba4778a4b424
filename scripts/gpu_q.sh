cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_quantiles.py -x -q --timeout 400 -p no:cacheprovider > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_q.log
