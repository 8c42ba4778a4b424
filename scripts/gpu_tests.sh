# full GPU test suite (no -x: every failure listed) + smoke
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/r02_gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02_smoke.log
grep -E "passed|failed|FAILED|exit" gpurun_out/r02_gpu_tests.log | tail -30; tail -2 gpurun_out/r02_smoke.log
