"""Per-phase timestamps of the d=1 kernel k_d1_lpc (GPM_D1_TIMING=1; %globaltimer of the
last launch of a CUDA graph of 20 back-to-back applies with fresh v; per phase: mean over
all warps of all CTAs of its end minus the earliest warp start, and the max).  Shapes from argv
(default 0); NU2 env (default 5)."""
import os, sys
os.environ["GPM_D1_TIMING"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
from bench import Applier
c = W.CONFIGS[2]
# (slot, name) in kernel order
SLOTS = [(8, "gdc.wait"), (7, "tab"), (9, "de.ready"), (1, "init"), (2, "u"), (3, "local"),
         (4, "publish"), (10, "scan"), (11, "recs"), (5, "fold.sync"), (13, "totals.sync"),
         (14, "carries"), (12, "corr"), (6, "out")]
shapes = [int(a) for a in sys.argv[1:]] or [0]
for n in (10000, 1000000):
    x = torch.from_numpy(W.config_points(c)[:n]).cuda()
    for shape in shapes:
        plan = g.Plan(x, g.Kernel(int(os.environ.get("NU2", "5")), c.ell))
        plan.set_option(1, shape)
        V = torch.randn((40, n), dtype=torch.float64, device="cuda")   # fresh v (> L2)
        VR = torch.stack([plan.to_rank(V[i]) for i in range(40)])
        O = torch.empty_like(V)
        for rank in (False, True):
            cs = torch.cuda.Stream()
            ap = Applier(g, plan, VR if rank else V, O, cs, rank_order=rank)
            for k in range(3):
                ap(k)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=cs):
                for k in range(20):
                    ap(k)
            with torch.cuda.stream(cs):
                graph.replay()
            torch.cuda.synchronize()
            mean = [plan.query(100 + s) / 1965.0 for s, _ in SLOTS]   # cycles -> us at 1965 MHz
            mx = [plan.query(200 + s) / 1965.0 for s, _ in SLOTS]
            print(f"n={n} shape={shape} rank={rank} end-of-phase us (mean/max):  " +
                  "  ".join(f"{nm}={m:.2f}/{M:.2f}" for (_, nm), m, M in zip(SLOTS, mean, mx)),
                  flush=True)
        plan.close()
