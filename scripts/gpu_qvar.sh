# A/B: quantiles on vs off, + quantile tests
cd $GRAFT_REPO_ROOT
: > gpurun_out/qvar.txt
run() { BB_LIB_PATH=$GRAFT_REPO_ROOT/paper_2412_04504_b200/$1 timeout 300 python bench.py --no-cpu-baseline --no-trace --reps 2000 --steps 2 --warmup 1 $2 > gpurun_out/qv.log 2>&1
  echo "$1 $2 $(python -c "import json; d=[json.loads(l) for l in open('gpurun_out/qv.log') if l.startswith('{')][0]; print('%.4e'%d['value'], d['roofline']['kernel_ms'])")" >> gpurun_out/qvar.txt; }
run libbinbatch_b200.so --no-quantiles
for v in $BB_VARIANTS; do run $v; done
run libbinbatch_b200.so
timeout 300 python -m pytest tests/test_gpu_quantiles.py -x -q -p no:cacheprovider >> gpurun_out/qvar.txt 2>&1
[ -n "$QPROF" ] && timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_kernel -c 1 -o gpurun_out/prof_genq4 python bench.py --reps 2000 --steps 1 --warmup 0 --no-cpu-baseline --no-trace > gpurun_out/ncu_genq.log 2>&1
true
