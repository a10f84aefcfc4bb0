"""Check that gp_kmvm calls captured in a CUDA graph compute the same result."""
import os, sys, ctypes
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
lib = g.load_library()
c = W.CONFIGS[2]
x = torch.from_numpy(W.config_points(c)[:200000]).cuda()
plan = g.Plan(x, g.Kernel(5, c.ell))
v = torch.randn(200000, dtype=torch.float64, device="cuda")
ref = plan.kmvm(v)
out = torch.zeros_like(v)
cs = torch.cuda.Stream()
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=cs):
    st = lib.gp_kmvm(plan._h, ctypes.c_void_p(v.data_ptr()), 1, ctypes.c_void_p(out.data_ptr()),
                     ctypes.c_void_p(cs.cuda_stream))
    print("status during capture", st, lib.gp_last_error())
print("capture status", torch.cuda.graphs.is_current_stream_capturing())
with torch.cuda.stream(cs):
    graph.replay()
torch.cuda.synchronize()
print("max diff after replay", float((out - ref).abs().max()), float(out.abs().max()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(cs):
    e0.record(cs); graph.replay(); e1.record(cs)
torch.cuda.synchronize()
print("replay ms", e0.elapsed_time(e1))
