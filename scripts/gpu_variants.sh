# A/B the fused kernel build variants on the same box
cd $GRAFT_REPO_ROOT
for v in libbinbatch_b200.so $BB_VARIANTS; do
  BB_LIB_PATH=$GRAFT_REPO_ROOT/paper_2412_04504_b200/$v timeout 300 python bench.py --steps 3 --warmup 2 --no-trace --no-cpu-baseline > gpurun_out/var_$v.log 2>&1
  echo "$v $(python -c "import json,sys; d=[json.loads(l) for l in open('gpurun_out/var_$v.log') if l.startswith('{')][0]; print('%.4e'%d['value'], d['roofline']['frac'])")" >> gpurun_out/variants.txt
done
