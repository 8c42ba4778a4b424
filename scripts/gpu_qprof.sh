cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/mem.txt
timeout 300 python bench.py --no-cpu-baseline --no-trace --reps 2000 --steps 2 --warmup 1 > gpurun_out/bq_on.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-trace --reps 2000 --steps 2 --warmup 1 --no-quantiles > gpurun_out/bq_off.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gen_kernel -c 1 -o gpurun_out/prof_genq python bench.py --reps 128 --steps 1 --warmup 0 --no-cpu-baseline --no-trace > gpurun_out/ncu_genq.log 2>&1
