cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_trace4.csv python scripts/trace_once.py > gpurun_out/ncu_trace_list.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"partition_kernel|request_kernel|binade|lindley_scan" -c 6 -o gpurun_out/prof_trace4 python scripts/trace_once.py > gpurun_out/ncu_trace2.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
