"""Headline counters per kernel of a --set full ncu capture:
python scripts/ncu_kernels.py <rep> [requests]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
reqs = float(sys.argv[2]) if len(sys.argv) > 2 else None
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].replace("bb::<unnamed>::", "")
    out = [name]
    for w in want:
        if w in d:
            out.append(f"{w.split('__')[1].split('.')[0]}={d[w]}{units[hdr.index(w)]}")
    st = sorted(((float(d[k].replace(',', '')), k) for k in hdr
                 if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")),
                reverse=True)[:3]
    out.append("stalls=" + ",".join(f"{k.split('stalled_')[1].split('_per')[0]}:{v:.2f}" for v, k in st))
    print("  ".join(out))
