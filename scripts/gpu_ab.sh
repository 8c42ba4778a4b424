# A/B on one box: the default library vs variants named in $VARIANTS (BB_LIB_PATH), reduced C3 sweep
if [ -n "$TESTS" ]; then timeout 900 python -m pytest $TESTS -x -q -p no:cacheprovider 2>&1 | tail -2; fi
for rep in 1 2; do
for lib in default $VARIANTS; do
  if [ "$lib" = default ]; then unset BB_LIB_PATH; else export BB_LIB_PATH=$PWD/paper_2412_04504_b200/$lib; fi
    timeout 600 python bench.py --reps ${REPS:-2000} --steps 3 --warmup 3 --no-cpu-baseline --no-trace --no-c5 --no-ab ${EXTRA:-} > gpurun_out/ab_$lib.log 2>&1
    python -c "
import json
for l in open('gpurun_out/ab_$lib.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$lib', 'value %.4g' % d['value'], 'kernel_ms %.1f' % d['roofline']['kernel_ms'])
"
  done
done
