"""Determinism / consistency check of the d=1 kernels: repeated applies bitwise equal,
rank order vs user order bitwise equal, for K and the lengthscale gradient."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2508_01864_b200 as g
import workloads as W

c = W.CONFIGS[2]
x = torch.from_numpy(W.config_points(c)).cuda()
V = torch.from_numpy(np.stack([W.config_vector(c, r) for r in range(3)])).cuda()
for two_nu in (3, 5):
    plan = g.Plan(x, g.Kernel(two_nu, c.ell))
    for grad in (False, True):
        f = (lambda v, **kw: plan.kmvm_dlengthscale(v, **kw)) if grad else None
        batch = plan.kmvm_dlengthscale(V) if grad else plan.kmvm(V)
        vr = plan.to_rank(V[1].contiguous())
        outs = []
        for rep in range(20):
            o = plan.kmvm_dlengthscale(vr, rank_order=True) if grad else plan.kmvm_rank(vr)
            outs.append(plan.from_rank(o))
        single_user = plan.kmvm_dlengthscale(V[1].contiguous()) if grad else plan.kmvm(V[1].contiguous())
        ndiff_rep = sum(int(not torch.equal(outs[0], o)) for o in outs)
        d_rank_batch = (outs[0] - batch[1]).abs().max().item()
        d_user_batch = (single_user - batch[1]).abs().max().item()
        d_rank_user = (outs[0] - single_user).abs().max().item()
        nbad = int((outs[0] != batch[1]).sum().item())
        print(f"2nu={two_nu} grad={grad}: rank repeats differing {ndiff_rep}/20; max|rank-batch| {d_rank_batch:.3e} "
              f"({nbad} entries); max|user-batch| {d_user_batch:.3e}; max|rank-user| {d_rank_user:.3e}; "
              f"scale {batch[1].abs().max().item():.3e}", flush=True)
    plan.close()
