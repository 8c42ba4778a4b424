"""Per-source-region instruction/sample breakdown of a --set full ncu capture
(needs --import-source and -lineinfo):  python scripts/ncu_lines.py <rep> <requests>"""
import collections
import csv
import io
import subprocess
import sys

rep, reqs = sys.argv[1], float(sys.argv[2])
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur = None
hdr = None
agg, samp = collections.Counter(), collections.Counter()
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 8 and r[0].isdigit():
        try:
            agg[(cur, int(r[0]))] += int(r[7])
            samp[(cur, int(r[0]))] += int(r[4])
        except ValueError:
            pass
tot, ts = sum(agg.values()), sum(samp.values())
print(f"lane-instr per request: {tot * 32 / reqs:.1f}")
byf = collections.Counter()
bys = collections.Counter()
for (f, l), v in agg.items():
    byf[f] += v
    bys[f] += samp[(f, l)]
for f, v in byf.most_common(6):
    print(f"  {f:28s} {v * 32 / reqs:6.1f} instr/req  {100 * bys[f] / ts:5.1f}% samples")
top = sorted(agg, key=lambda k: -agg[k])[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]
for k in top:
    print(f"  {agg[k] * 32 / reqs:5.1f} instr/req {100 * samp[k] / ts:5.1f}% samples  {k[0]}:{k[1]}")
