"""PCIe copy throughput on the GPU box: 8 MB pinned H2D alone, D2H alone, both at once
(two streams) -- the ceiling of bench.py's host-buffer e2e number."""
import time
import torch
n = 1_000_000
K = 40
h_in = [torch.randn(n, dtype=torch.float64).pin_memory() for _ in range(4)]
h_out = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(4)]
d = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(4)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(mode):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(K):
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s1):
                d[k % 2].copy_(h_in[k % 4], non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s2):
                h_out[k % 4].copy_(d[2 + k % 2], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / K
    print(f"{mode}: {dt * 1e6:.1f} us per 8 MB ({8e6 / dt / 1e9:.1f} GB/s per direction)", flush=True)
for m in ("h2d", "d2h", "both", "h2d", "d2h", "both"):
    run(m)
