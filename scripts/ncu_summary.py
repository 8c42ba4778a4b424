"""Summarise ncu captures into profiles/ (tracked).

  python scripts/ncu_summary.py launches <launches.csv> <out.md>
  python scripts/ncu_summary.py full <report.ncu-rep> <out.json> [requests_per_launch]

`launches`: per-kernel share of the device time from a
`--metrics gpu__time_duration.sum` launch list (cold-cache, serialised: use
the shares, not the absolutes).  `full`: the headline counters of a
`--set full` capture (duration, DRAM bytes, issue activity, stall reasons,
instructions per request when the request count is given).
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
        name = d["Kernel Name"].split("(")[0].replace("bb::<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    lines = [f"# kernel launch list: {path}", "",
             "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]


def full(path, out, requests=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")].split("(")[0].replace("bb::<unnamed>::", "")}
        for m in WANT:
            if m in hdr:
                d[m] = row[hdr.index(m)] + (" " + units[hdr.index(m)] if units[hdr.index(m)] else "")
        stalls = {}
        for i, m in enumerate(hdr):
            if m.startswith("smsp__average_warps_issue_stalled_") and m.endswith("per_issue_active.ratio"):
                try:
                    v = float(row[i])
                except ValueError:
                    continue
                if v >= 0.1:
                    stalls[m[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
        try:
            rd = float(row[hdr.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(row[hdr.index("dram__bytes_write.sum")].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            d["dram_bytes_per_launch"] = rd * scale.get(units[hdr.index("dram__bytes_read.sum")], 1) + \
                wr * scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
        except (ValueError, KeyError):
            pass
        if requests:
            inst = float(row[hdr.index("smsp__inst_executed.sum")].replace(",", ""))
            d["warp_instructions_per_request_step"] = inst * 32 / float(requests)
            if "dram_bytes_per_launch" in d:
                d["dram_bytes_per_request"] = d["dram_bytes_per_launch"] / float(requests)
            d["requests_per_launch"] = float(requests)
        res.append(d)
    json.dump(res if len(res) > 1 else res[0], open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None)
