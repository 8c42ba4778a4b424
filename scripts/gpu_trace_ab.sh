# trace-mode A/B on one box: the default library vs variants named in $VARIANTS (BB_LIB_PATH), C2 timing
if [ -n "$TESTS" ]; then timeout 900 python -m pytest $TESTS -x -q -p no:cacheprovider 2>&1 | tail -2; fi
for rep in 1 2 3; do
for lib in default $VARIANTS; do
  if [ "$lib" = default ]; then unset BB_LIB_PATH; else export BB_LIB_PATH=$PWD/paper_2412_04504_b200/$lib; fi
  timeout 600 python scripts/trace_bench.py > gpurun_out/tab_$lib.log 2>&1
  python -c "
import json
for l in open('gpurun_out/tab_$lib.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$lib', 'ms %.4f' % d['ms_per_run'], 'part_ms %.4f' % d['roofline']['kernel_ms'])
" || tail -5 gpurun_out/tab_$lib.log
done
done
