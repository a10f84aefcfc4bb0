"""Summarise an ncu --csv launch list: count and total time per kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if r and r[0] == 'ID':
        hdr = r; start = i; break
data = rows[start + 1:]
ki = hdr.index('Kernel Name'); mi = hdr.index('Metric Name'); vi = hdr.index('Metric Value'); ii = hdr.index('ID')
per = collections.defaultdict(dict)
for r in data:
    per[int(r[ii])][r[mi]] = (r[ki], float(r[vi].replace(',', '')))
agg = collections.defaultdict(lambda: [0, 0.0])
for i, m in per.items():
    name, t = m['gpu__time_duration.sum']
    short = name.split('(')[0]
    short = short[-70:]
    agg[short][0] += 1; agg[short][1] += t
tot = sum(t for _, t in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"  {c:5d} {t/1e3:10.1f} us ({100*t/tot:5.1f}%) avg {t/c/1e3:8.1f} us  {k}")
