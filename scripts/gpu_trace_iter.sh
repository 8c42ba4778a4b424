# trace-mode iteration: exactness tests, the C2 timing, a launch list and a full capture of the C2 kernels
timeout 900 python -m pytest tests/test_gpu_trace_graph.py tests/test_gpu_trace.py tests/test_gpu_reference_rng.py -x -q -p no:cacheprovider > gpurun_out/r02_trace_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r02_trace_tests.log
tail -3 gpurun_out/r02_trace_tests.log
timeout 600 python scripts/trace_bench.py > gpurun_out/r02_trace_bench.log 2>&1; echo "trace bench exit $?"
tail -c 1200 gpurun_out/r02_trace_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_trace_launches.csv python scripts/trace_c2_once.py 1 > /dev/null 2>&1
python scripts/ncu_summary.py launches gpurun_out/r02_trace_launches.csv gpurun_out/r02_trace_launches.md | head -40
if [ -n "$FULL" ]; then timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$FULL" -c 8 -o gpurun_out/r02_trace_full python scripts/trace_c2_once.py 1 > gpurun_out/r02_trace_full.log 2>&1; echo "ncu full $?"; fi
