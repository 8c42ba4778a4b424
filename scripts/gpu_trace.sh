cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_trace5.csv python scripts/trace_once.py > gpurun_out/ncu_trace_list.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"partition_kernel|request_kernel|binade|lindley_scan" -c 6 -o gpurun_out/prof_trace5 python scripts/trace_once.py > gpurun_out/ncu_trace2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_kernel -c 1 -o gpurun_out/prof_gen5 python bench.py --reps 1500 --steps 1 --warmup 0 --no-cpu-baseline --no-trace > gpurun_out/ncu_gen.log 2>&1
