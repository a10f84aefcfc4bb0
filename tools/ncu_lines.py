"""Per-CUDA-line hot spots from an ncu report (ncu --page source --print-source cuda,sass)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
filt = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
path = fn = None
hdr = None
agg = collections.defaultdict(lambda: collections.Counter())
text = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        fn = r[1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        if filt and filt not in fn:
            continue
        key = (fn, path, int(r[0]))
        text[key] = r[1]
        agg[key]["stall"] += int(r[4] or 0)
        agg[key]["inst"] += int(r[7] or 0)
fns = sorted({k[0] for k in agg})
for f in fns:
    items = [(k, v) for k, v in agg.items() if k[0] == f]
    ts = sum(v["stall"] for _, v in items) or 1
    ti = sum(v["inst"] for _, v in items) or 1
    print(f"== {f[:100]}  samples {ts}  warp-instr {ti}")
    for k, v in sorted(items, key=lambda kv: -kv[1]["stall"])[:top]:
        print(f"  {100 * v['stall'] / ts:5.1f}% st {100 * v['inst'] / ti:5.1f}% in  "
              f"{k[1]}:{k[2]:<5d} {text[k].strip()[:70]}")
