cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_kernel -c 1 -o gpurun_out/prof_genq3 python bench.py --reps 2000 --steps 1 --warmup 0 --no-cpu-baseline --no-trace > gpurun_out/ncu_genq.log 2>&1
