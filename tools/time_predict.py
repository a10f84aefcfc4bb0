"""Wall time of config-5 posterior mean (union setup on first call) and of setups."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2508_01864_b200 as g
import workloads as W
c5 = W.CONFIGS[5]
x = W.config_points(c5); y = W.config_response(c5, x)
dev = torch.device("cuda")
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    plan = g.Plan(torch.from_numpy(x).to(dev), g.Kernel(3, c5.ell, form=g.FORM_PRODUCT))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    z = torch.from_numpy(W.config_queries(c5)).to(dev)
    alpha = torch.randn(x.shape[0], dtype=torch.float64, device=dev)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    mu = plan.predict(z, alpha, [1.0, 0.5, -0.3])
    torch.cuda.synchronize(); t3 = time.perf_counter()
    mu = plan.predict(z, alpha, [1.0, 0.5, -0.3])
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"rep {rep}: setup {t1-t0:.4f} s, predict (incl. union setup) {t3-t2:.4f} s, again {t4-t3:.4f} s", flush=True)
    plan.close()
