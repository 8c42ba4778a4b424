# iterate: GPU tests, bench, one ncu capture of the fused kernel at full occupancy
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_kernel -c 1 -o gpurun_out/prof_gen4 python bench.py --reps 1500 --steps 1 --warmup 0 --no-cpu-baseline --no-trace > gpurun_out/ncu_gen.log 2>&1
