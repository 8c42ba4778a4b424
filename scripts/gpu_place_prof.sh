# place_kernel / count_kernel source-level capture on the C2 trace (summaries only come back)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_trace.py tests/test_gpu_trace_graph.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python scripts/trace_bench.py 2>&1 | cut -c1-400
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KERN:-place_kernel}" -c ${NK:-1} -o gpurun_out/place python scripts/trace_c2_once.py 1 > /dev/null 2>&1; echo "ncu rc=$?"
python scripts/ncu_lines.py gpurun_out/place.ncu-rep 1e7 > gpurun_out/place_lines.txt
python scripts/ncu_summary.py full gpurun_out/place.ncu-rep gpurun_out/place_ncu.json 1e7
rm -f gpurun_out/place.ncu-rep
head -40 gpurun_out/place_lines.txt
python -c "import json;d=json.load(open('gpurun_out/place_ncu.json'));print(json.dumps(d)[:1500])"
