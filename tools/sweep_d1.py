"""Time the d=1 single-chunk apply k_d1_lpc (CUDA graph of 100 back-to-back applies, fresh
v each, config 2) for the thread-block shapes given on the command line (default: all):
single column in user and rank order, and 16 columns per call (multi-RHS, per MVM).
Each shape's output is compared with shape 0's on the same v (relative max difference)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ctypes
import torch
import paper_2508_01864_b200 as g
import workloads as W
from bench import Applier, time_graph

shapes = [int(a) for a in sys.argv[1:]] or [0, 1, 2]
c = W.CONFIGS[2]
x = torch.from_numpy(W.config_points(c)).cuda()
nv = 100
V = torch.randn((nv, c.n), dtype=torch.float64, device="cuda")
O = torch.empty_like(V)
lib = g.load_library()


class Multi:
    """gp_kmvm / gp_kmvm_rank with 16 columns per call (V[16k .. 16k+15])."""
    def __init__(self, plan, VV, s, rank):
        self.f = lib.gp_kmvm_rank if rank else lib.gp_kmvm
        self.h, self.VV, self.s = plan._h, VV, ctypes.c_void_p(s.cuda_stream)
    def __call__(self, k):
        b = 16 * (k % 6)
        st = self.f(self.h, ctypes.c_void_p(self.VV[b].data_ptr()), 16,
                    ctypes.c_void_p(O[b].data_ptr()), self.s)
        assert st == 0


for two_nu in (5, 3):
    plan = g.Plan(x, g.Kernel(two_nu, c.ell))
    VR = torch.stack([plan.to_rank(V[i]) for i in range(nv)])
    plan.set_option(1, 0)
    ref_u = plan.kmvm(V[3]).clone()
    ref_r = plan.kmvm_rank(VR[3]).clone()
    for shape in shapes:
        plan.set_option(1, shape)
        eu = (plan.kmvm(V[3]) - ref_u).abs().max().item() / ref_u.abs().max().item()
        er = (plan.kmvm_rank(VR[3]) - ref_r).abs().max().item() / ref_r.abs().max().item()
        row = dict(two_nu=two_nu, shape=shape, relerr_user=eu, relerr_rank=er)
        for rank in (False, True):
            res = time_graph(lambda s: Applier(g, plan, VR if rank else V, O, s, rank_order=rank),
                             100, 5, 1, reps=5, stats={})
            row["us_rank" if rank else "us_user"] = res[0] / 100 * 1e6
            res = time_graph(lambda s: Multi(plan, VR if rank else V, s, rank), 12, 3, 1, reps=3,
                             stats={})
            row["us_rank16" if rank else "us_user16"] = res[0] / (12 * 16) * 1e6
        print(json.dumps(row), flush=True)
    plan.close()
