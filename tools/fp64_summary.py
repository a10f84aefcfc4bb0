"""FP64 work and DRAM bytes per apply from an ncu --csv metrics log (tools/gpu/fp64.sh):
per apply-path kernel, thread-level DFMA/DADD/DMUL -> FLOPs (DFMA = 2), duration, GFLOP/s."""
import collections
import csv
import sys

APPLY = ("k_d1_lpc", "k_d1_big", "k_cp_carry", "k_pack", "k_low2", "k_low3", "k_mid3", "k_cp", "k_epilogue")


def summary(path, applies):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi, ii = (hdr.index(h) for h in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    for r in rows[start + 1:]:
        per[int(r[ii])][r[mi]] = (r[ki], float(r[vi].replace(",", "")))
    agg = collections.defaultdict(lambda: collections.Counter())
    for m in per.values():
        name = m["gpu__time_duration.sum"][0].split("(")[0].replace("void ", "").replace("gpm::", "")
        if not any(a in name for a in APPLY):
            continue
        c = agg[name]
        c["n"] += 1
        c["ns"] += m["gpu__time_duration.sum"][1]
        c["flop"] += (2 * m["sm__sass_thread_inst_executed_op_dfma_pred_on.sum"][1]
                      + m["sm__sass_thread_inst_executed_op_dadd_pred_on.sum"][1]
                      + m["sm__sass_thread_inst_executed_op_dmul_pred_on.sum"][1])
        c["dram"] += m["dram__bytes_read.sum"][1] + m["dram__bytes_write.sum"][1]
    tot = collections.Counter()
    print(f"{path}: per apply ({applies} applies profiled)")
    for name, c in sorted(agg.items(), key=lambda x: -x[1]["ns"]):
        tot.update(c)
        print(f"  {name[:60]:60s} {c['ns'] / applies / 1e3:9.1f} us  {c['flop'] / applies / 1e9:8.3f} GFLOP"
              f"  {c['flop'] / c['ns']:8.1f} GFLOP/s  {c['dram'] / applies / 1e6:8.1f} MB DRAM")
    print(f"  {'total (serialised)':60s} {tot['ns'] / applies / 1e3:9.1f} us  "
          f"{tot['flop'] / applies / 1e9:8.3f} GFLOP  {tot['flop'] / tot['ns']:8.1f} GFLOP/s  "
          f"{tot['dram'] / applies / 1e6:8.1f} MB DRAM")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        summary(p, 2)
