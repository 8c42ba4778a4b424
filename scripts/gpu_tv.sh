# GPU tests, then A/B of the fused-kernel build variants ($BB_VARIANTS)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
rm -f gpurun_out/variants.txt
BB_VARIANTS="$BB_VARIANTS" bash scripts/gpu_variants.sh
