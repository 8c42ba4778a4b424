cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_quantiles.py -x -q --timeout 400 -p no:cacheprovider > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
timeout 300 python bench.py --no-cpu-baseline --no-trace --reps 2000 --steps 2 --warmup 1 > gpurun_out/bq_on.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gen_kernel -c 1 -o gpurun_out/prof_genq2 python bench.py --reps 512 --steps 1 --warmup 0 --no-cpu-baseline --no-trace > gpurun_out/ncu_genq.log 2>&1
