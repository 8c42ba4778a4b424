# quick quantile-mode timing: a reduced C3 sweep (2000 replications/point), kernel ms only
timeout 600 python bench.py --reps 2000 --steps 3 --warmup 3 --no-cpu-baseline --no-trace --no-c5 --no-ab > gpurun_out/r02_qq.log 2>&1; echo "bench exit $?"
python - <<'P'
import json
for l in open("gpurun_out/r02_qq.log"):
    if l.startswith("{"):
        d=json.loads(l); print("value", d["value"], "kernel_ms", d["roofline"]["kernel_ms"], "ms_per_step", d["ms_per_step"])
P
