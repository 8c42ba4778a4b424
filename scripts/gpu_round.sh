# smoke + gpu tests + default bench + reference arm + launch list + full capture of gen_kernel
cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/smi.txt 2>&1; nproc >> gpurun_out/smi.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_default.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --reps 256 --steps 1 --warmup 1 --no-cpu-baseline --no-ab > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_kernel -c 1 -o gpurun_out/prof_genq python bench.py --reps 2000 --steps 1 --warmup 0 --no-cpu-baseline --no-trace --no-ab > gpurun_out/ncu_genq.log 2>&1
