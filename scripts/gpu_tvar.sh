# A/B: trace pipeline variants (C2 10^7 run, bench trace leg)
cd $GRAFT_REPO_ROOT
: > gpurun_out/tvar.txt
for v in libbinbatch_b200.so $BB_VARIANTS; do
  BB_LIB_PATH=$GRAFT_REPO_ROOT/paper_2412_04504_b200/$v timeout 300 python bench.py --reps 8 --steps 1 --warmup 1 --no-cpu-baseline --no-ab --no-c5 > gpurun_out/tv.log 2>&1
  echo "$v $(python -c "import json; d=[json.loads(l) for l in open('gpurun_out/tv.log') if l.startswith('{')][0]['trace']; print(d['ms_per_run'], d['roofline']['kernel_ms'], d['bit_exact_vs_reference_run'])")" >> gpurun_out/tvar.txt
done
