"""Profiling driver: set up one config and run a few applies (for ncu / timing)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_2508_01864_b200 as g
import workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--nu2", type=int, default=5)
ap.add_argument("--applies", type=int, default=5)
ap.add_argument("--form", type=int, default=0)
ap.add_argument("--rank", action="store_true")
ap.add_argument("--nrhs", type=int, default=1)
ap.add_argument("--shape", type=int, default=-1)
args = ap.parse_args()
c = W.CONFIGS[args.config]
x = torch.from_numpy(W.config_points(c)).cuda()
plan = g.Plan(x, g.Kernel(args.nu2, c.ell, form=args.form))
if args.shape >= 0:
    plan.set_option(1, args.shape)
def _vec(r):
    a = np.stack([W.config_vector(c, r * args.nrhs + j) for j in range(args.nrhs)])
    return torch.from_numpy(a[0] if args.nrhs == 1 else a).cuda()


V = [_vec(r) for r in range(min(args.applies, 8))]
if os.environ.get('GPM_PROF_TIMING'):
    pass
out = torch.empty_like(V[0])
for k in range(args.applies):
    if args.rank:
        plan.kmvm_rank(V[k % len(V)], out)
    else:
        plan.kmvm(V[k % len(V)], out)
torch.cuda.synchronize()
print("ok", plan.launches_per_apply, plan.model_bytes)
