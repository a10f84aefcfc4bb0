"""Per-phase timestamps of the d=1 fast kernel (GPM_D1_TIMING=1)."""
import os, sys
os.environ["GPM_D1_TIMING"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
c = W.CONFIGS[2]
names = ["tma+load", "pass1", "scan", "grid.sync", "carries", "pass2+store"]
for n in (10000, 1000000):
    x = torch.from_numpy(W.config_points(c)[:n]).cuda()
    for shape in (int(os.environ.get("GPM_D1_SHAPE", "2")),):
        plan = g.Plan(x, g.Kernel(int(os.environ.get("NU2", "5")), c.ell))
        plan.set_option(1, shape)
        V = torch.randn((64, n), dtype=torch.float64, device="cuda")   # fresh v (> L2)
        vr = plan.to_rank(V[0])
        for rank in (False, True):
            for k in range(5):
                (plan.kmvm_rank(vr) if rank else plan.kmvm(V[k]))
            torch.cuda.synchronize()
            st = [plan.query(8 + k) for k in range(6)]
            parts = [f"{nm}={(st[i] - (st[i-1] if i else 0)) / 1e3:.2f}" for i, nm in enumerate(names)]
            parts.append(f"total={st[-1]/1e3:.2f}")
            mx = [plan.query(20 + k) for k in range(6)]
            parts.append("| max: " + " ".join(f"{nm}={m/1e3:.2f}" for nm, m in zip(names, mx)))
            print(f"n={n} shape={shape} rank={rank} " + " ".join(parts), flush=True)
