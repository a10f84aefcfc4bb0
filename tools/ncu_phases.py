"""Warp-stall samples of k_d1_lpc bucketed by kernel phase: the SASS is cut at the
%globaltimer reads of the LPC_STAMP macros (present in the binary whether or not timing is
enabled), in address order.  python tools/ncu_phases.py REPORT.ncu-rep"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = next(r for r in rows if "Address" in r and "Source" in r)
ai, si, ni = hdr.index("Address"), hdr.index("Source"), hdr.index("# Samples")
stall_cols = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
ie = hdr.index("Instructions Executed") if "Instructions Executed" in hdr else None
phase = 0
agg = defaultdict(lambda: [0, defaultdict(int), 0, 0])
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= ni:
        continue
    src = r[si]
    try:
        s = int(float(r[ni] or 0))
    except ValueError:
        continue
    if "GLOBALTIMER" in src:
        phase += 1
    a = agg[phase]
    a[0] += s
    a[2] += 1
    if ie is not None:
        try:
            a[3] += int(float(r[ie] or 0))
        except ValueError:
            pass
    for i, name in stall_cols:
        try:
            a[1][name] += int(float(r[i] or 0))
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values())
print(f"total samples {tot}")
for p in sorted(agg):
    s, st, ninst, nexec = agg[p]
    top = sorted(st.items(), key=lambda kv: -kv[1])[:5]
    print(f"after stamp #{p:2d}: {s:6d} samples ({100.0 * s / max(tot, 1):5.1f}%), {ninst:4d} SASS, "
          f"{nexec:9d} warp-inst  " + " ".join(f"{k}={v}" for k, v in top))
