"""Apply time of configs 3 / 4 for near-field block sizes (env GPM_NEAR_LB=lb2,lb3,lb3m)."""
import os, sys, json, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
cfg = int(sys.argv[1]); nu2 = int(sys.argv[2]); form = int(sys.argv[3]) if len(sys.argv) > 3 else 0
c = W.CONFIGS[cfg]
x = torch.from_numpy(W.config_points(c)).cuda()
plan = g.Plan(x, g.Kernel(nu2, c.ell, form=form))
v = torch.randn(c.n, dtype=torch.float64, device="cuda")
out = plan.kmvm(v)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10 if cfg == 4 else 30
e0.record()
for _ in range(reps):
    plan.kmvm(v, out)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"cfg": cfg, "nu2": nu2, "form": form, "lb": os.environ.get("GPM_NEAR_LB", "default"),
                  "ms": e0.elapsed_time(e1) / reps, "launches": plan.launches_per_apply}), flush=True)
