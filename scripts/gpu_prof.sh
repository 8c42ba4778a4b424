# tests + launch list + full ncu capture of the two dominant kernels
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --reps 256 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gen_kernel -c 1 -o gpurun_out/prof_gen python bench.py --reps 128 --steps 1 --warmup 0 --no-cpu-baseline --no-trace > gpurun_out/ncu_gen.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"partition_kernel|lindley|request_kernel" -c 4 -o gpurun_out/prof_trace python scripts/trace_once.py > gpurun_out/ncu_trace.log 2>&1
timeout 300 python bench.py --reps 10000 --steps 3 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
