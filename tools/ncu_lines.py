"""Per-source-line warp-stall samples of one kernel in an ncu report (needs -lineinfo and
--import-source on):  python tools/ncu_lines.py REPORT.ncu-rep [min_samples]
Prints file:line, samples, the dominant stall reasons and the source text, in file order,
plus per-file totals."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
mn = int(sys.argv[2]) if len(sys.argv) > 2 else 10
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
cur_file = "?"
agg = defaultdict(lambda: [0, defaultdict(int), ""])
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        s = int(float(r[hdr.index("# Samples")] or 0))
    except ValueError:
        continue
    key = (cur_file, int(r[0]))
    agg[key][0] += s
    agg[key][2] = r[1]
    for k, v in zip(hdr, r):
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                agg[key][1][k[6:]] += int(float(v or 0))
            except ValueError:
                pass
tot = sum(v[0] for v in agg.values())
print(f"total samples {tot}")
per_file = defaultdict(int)
for (f, ln), (s, st, src) in sorted(agg.items()):
    per_file[f] += s
    if s >= mn:
        top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        print(f"{f}:{ln:<5d} {s:6d}  {','.join(f'{k}={v}' for k, v in top):45s} {src.strip()[:70]}")
print(dict(per_file))
