# round-end evidence: the default bench line, the reference arm, launch lists and full ncu captures
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/r02_bench_default.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/r02_bench_default.log | tail -1 > gpurun_out/r02_bench_default.json
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_reference.log 2>&1; echo "ref rc=$?"
grep '^{' gpurun_out/r02_bench_reference.log | tail -1 > gpurun_out/r02_bench_reference.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_bench_launches.csv python bench.py --reps 256 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_kernel -c 1 -o gpurun_out/r02_genq_full python bench.py --reps 2000 --steps 1 --warmup 0 --no-cpu-baseline --no-trace --no-ab --no-c5 > /dev/null 2>&1; echo "genq rc=$?"
BB_WARP_MODE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:genw_kernel -c 1 -o gpurun_out/r02_genw_full python scripts/warp_probe.py > /dev/null 2>&1; echo "genw rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"count_kernel|tscan_kernel|place_kernel|request_kernel|lindley_scan|binade_scan|binade_chain|sel_hist_kernel|sel_collect" -c 12 -o gpurun_out/r02_trace_full python scripts/trace_c2_once.py 1 > /dev/null 2>&1; echo "trace rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_trace_launches.csv python scripts/trace_c2_once.py 1 > /dev/null 2>&1; echo "trace launches rc=$?"
# summaries on the box (the .ncu-rep files exceed gpurun's 64 MiB copy-back)
python scripts/ncu_summary.py launches gpurun_out/r02_bench_launches.csv gpurun_out/r02_bench_launches.md > /dev/null
python scripts/ncu_summary.py launches gpurun_out/r02_trace_launches.csv gpurun_out/r02_trace_c2_launches.md > /dev/null
python scripts/ncu_summary.py full gpurun_out/r02_genq_full.ncu-rep gpurun_out/r02_gen_kernel_q_ncu.json 2.1e10
python scripts/ncu_lines.py gpurun_out/r02_genq_full.ncu-rep 2.1e10 > gpurun_out/r02_gen_kernel_q_lines.txt
python scripts/ncu_summary.py full gpurun_out/r02_genw_full.ncu-rep gpurun_out/r02_genw_kernel_ncu.json 4.736e9
python scripts/ncu_summary.py full gpurun_out/r02_trace_full.ncu-rep gpurun_out/r02_trace_c2_ncu.json 1e7
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out | tail -16
cat gpurun_out/r02_bench_default.json | cut -c1-1500
