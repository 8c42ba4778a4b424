# round-2 GPU check: the full -m gpu suite (incl. the reference's own C++ suites)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/r2_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2_gpu_tests.log
tests/cpp/_bin/acceptance_b200 > gpurun_out/r2_acceptance.log 2>&1; echo "rc=$?" >> gpurun_out/r2_acceptance.log
tests/cpp/_bin/unit_tests_b200 > gpurun_out/r2_unit.log 2>&1; echo "rc=$?" >> gpurun_out/r2_unit.log
