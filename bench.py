#!/usr/bin/env python
"""bench.py -- the BASELINE.json metric on B200: kernel MVMs/s (and HBM GB/s as a fraction
of the measured roofline) of the exact fast Matern K.v at N = 1e6, d = 1 (configs[1]),
plus d = 2 / d = 3 applies (configs[2], configs[3]) and the config-5 CG solve time as
extra fields.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--no-cg] [--no-graph] [--no-extras] [--no-cpu]

One "step" = one K.v apply of config 2 (d = 1, N = 1e6, nu = 5/2, l = 0.05, x ~ N(0,1))
with a fresh v, through the C ABI (gp_kmvm), the structure set up once (as configs[1]
says).  The K timed applies are captured as one CUDA graph of gp_kmvm calls and replayed
once (device time by CUDA events); the plain stream-loop time is reported beside it.  Inputs are larger than L2: the steps cycle through 100 distinct v / out buffers
(1.6 GB).  value = applies of all ranks / max-over-ranks device time.  Multi-GPU runs
are independent replicas (each rank its own plan and inputs; no data-path collective:
DESIGN.md "Multi-GPU"), so scaling is weak.

--impl reference times the CPU oracle (oracle/, dense O(N^2), all host cores) on the
same workload, each step a bounded sample of rows, extrapolated to whole MVMs.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "ncu_traffic.json")
FALLBACK_HBM = 6650.0


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def d1_kernel_name(shape, user=True):
    """Name of the d = 1 kernel (nu = 5/2) of a plan's thread-block shape (gp_plan_set_option
    option 1): k_d1_lpc<P, KIND, threads, segments, points per segment, user order>."""
    u = "user" if user else "rank"
    shapes = {0: f"k_d1_lpc<2,0,256,3,9,{u}>", 1: f"k_d1_lpc<2,0,256,3,10,{u}>",
              2: f"k_d1_lpc<2,0,256,4,7,{u}>"}
    return shapes.get(shape, f"d1 shape {shape}")


def ncu_traffic(key):
    try:
        with open(TRAFFIC_PATH) as f:
            return json.load(f).get(key)
    except Exception:
        return None


class ClockSampler:
    """Samples SM clock + throttle reasons with NVML while the timed region runs."""

    REASONS = {
        0x0000000000000001: "gpu_idle", 0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap", 0x0000000000000008: "hw_slowdown",
        0x0000000000000010: "sync_boost", 0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown", 0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- helpers

def dist_setup():
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(val: float, ws: int) -> float:
    if ws == 1:
        return val
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([val], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(val: float, ws: int) -> float:
    if ws == 1:
        return val
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([val], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


class Applier:
    """Pre-marshalled gp_kmvm calls (no per-call Python tensor work in the timed loop)."""

    def __init__(self, g, plan, V, OUT, stream, rank_order=False, grad=False):
        lib = g.load_library()
        if grad:   # lengthscale-gradient MVM (gp_kmvm_dlengthscale)
            ro = 1 if rank_order else 0
            self.f = lambda h, v, k, o, s: lib.gp_kmvm_dlengthscale(h, v, k, o, ro, s)
        else:
            self.f = lib.gp_kmvm_rank if rank_order else lib.gp_kmvm
        self.h = plan._h
        self.vp = [ctypes.c_void_p(V[i].data_ptr()) for i in range(V.shape[0])]
        self.op = [ctypes.c_void_p(OUT[i].data_ptr()) for i in range(OUT.shape[0])]
        self.s = ctypes.c_void_p(stream.cuda_stream)
        self.nv = V.shape[0]

    def __call__(self, k):
        st = self.f(self.h, self.vp[k % self.nv], 1, self.op[k % self.nv], self.s)
        if st:
            raise RuntimeError("gp_kmvm failed")


def time_applies(applier, steps, warmup, stream, ws):
    """Returns (seconds for `steps` applies, max over ranks, per-launch mean seconds)."""
    import torch
    for k in range(warmup):
        applier(k)
    torch.cuda.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(steps):
        applier(warmup + k)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    sec = e0.elapsed_time(e1) / 1e3
    return max_over_ranks(sec, ws), sec


def time_graph(make_applier, steps, warmup, ws, reps=1, stats=None):
    """Capture `steps` applies in one CUDA graph (on a side stream) and time `reps` replays
    (each bracketed by barrier + synchronize); returns the median replay as (max-over-ranks
    seconds, local seconds) or None if capture is unsupported.  stats (dict) receives the
    per-apply p10 / p50 / p90 over the replays (SURVEY §8(d) timing protocol)."""
    import torch
    cs = torch.cuda.Stream()
    try:
        ap = make_applier(cs)
        for k in range(warmup):
            ap(k)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cs):
            for k in range(steps):
                ap(k)
        with torch.cuda.stream(cs):
            graph.replay()          # warm replay (replay() launches on the current stream)
        torch.cuda.synchronize()
    except Exception as e:          # pragma: no cover - reported in the JSON line
        print(f"graph capture failed: {e}", file=sys.stderr)
        return None
    secs = []
    for _ in range(reps):
        barrier(ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(cs):
            e0.record(cs)
            graph.replay()
            e1.record(cs)
        torch.cuda.synchronize()
        barrier(ws)
        secs.append(max_over_ranks(e0.elapsed_time(e1) / 1e3, ws))
    order = sorted(secs)
    med = order[len(order) // 2]
    if stats is not None:
        q = lambda f: order[min(len(order) - 1, int(f * (len(order) - 1) + 0.5))] / steps * 1e3
        stats.update({"replays": reps, "apply_ms_p10": q(0.1), "apply_ms_p50": q(0.5),
                      "apply_ms_p90": q(0.9)})
    return med, med


def per_launch(applier, steps, stream):
    """Mean device duration of one apply (events bracketing each launch)."""
    import torch
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for k, (a, b) in enumerate(evs):
        a.record(stream)
        applier(k)
        b.record(stream)
    torch.cuda.synchronize()
    d = [a.elapsed_time(b) / 1e3 for a, b in evs]
    return statistics.mean(d), statistics.median(d), min(d)


# ----------------------------------------------------------------------------- our arm

def run_ours(args, ws, rank, local):
    import torch
    import paper_2508_01864_b200 as g
    g.load_library()
    # plan / scratch allocations through PyTorch's caching allocator (gp_set_allocator):
    # setups after the first reuse cached blocks instead of cudaMalloc / cudaFree
    g.use_torch_allocator()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    cfg = W.CONFIGS[2]
    n = cfg.n
    x = torch.from_numpy(W.config_points(cfg)).to(dev)
    nv = 100
    # 100 distinct v (and out) buffers: 1.6 GB > 126 MB L2
    V = torch.empty((nv, n), dtype=torch.float64, device=dev)
    for r in range(nv):
        V[r] = torch.from_numpy(W.config_vector(cfg, r + 100 * rank))
    OUT = torch.empty_like(V)
    hbm, peak_kind = peaks()
    result = {}
    # process warm-up outside any timed region: the first plan of a process pays CUDA's lazy
    # module loading of the library's kernels and the allocator's pool growth
    wp = g.Plan(x[:4096].contiguous(), g.Kernel(5, cfg.ell), stream)
    wp.kmvm(V[0, :4096].contiguous())
    wp.close()
    torch.cuda.synchronize()

    def measure(two_nu, steps, warmup, sampler=None, vin=None, rank_order=False, reps=1):
        torch.cuda.synchronize()
        t_setup = time.perf_counter()
        plan = g.Plan(x, g.Kernel(two_nu, cfg.ell), stream)
        torch.cuda.synchronize()
        t_setup = time.perf_counter() - t_setup
        gstats = {"setup_s": t_setup}
        VV = V if vin is None else vin(plan)
        ap = Applier(g, plan, VV, OUT, stream, rank_order=rank_order)
        mk = lambda st: Applier(g, plan, VV, OUT, st, rank_order=rank_order)
        import contextlib
        with (sampler if sampler else contextlib.nullcontext()):
            gr = None if args.no_graph else time_graph(mk, steps, warmup, ws, reps, gstats)
            if gr is None:
                sec_max, sec = time_applies(ap, steps, warmup, stream, ws)
            else:
                sec_max, sec = gr
        loop_max, _ = time_applies(ap, min(steps, 500), 3, stream, ws)
        mean_l, med_l, min_l = per_launch(ap, min(steps, 200), stream)
        info = {"graph": gr is not None, "stream_loop_ms_per_step": loop_max / min(steps, 500) * 1e3,
                **gstats}
        return plan, ap, sec_max, sec, mean_l, med_l, min_l, info

    sampler = ClockSampler(local)
    two_nu = 5
    plan, ap, sec_max, sec, mean_l, med_l, min_l, tinfo = measure(two_nu, args.steps, args.warmup,
                                                                   sampler, reps=5)
    total = sum_over_ranks(args.steps, ws)
    value = total / sec_max
    model_bytes = plan.model_bytes
    launches = plan.launches_per_apply
    # average launch duration of the dominant (only) kernel over the timed region: the graph
    # replay holds exactly K back-to-back launches of it (CUDA events on the replay stream);
    # the per-launch event brackets (launch_ms_isolated) include the event gaps
    launch_s = sec / args.steps if tinfo["graph"] else mean_l
    achieved = model_bytes / launch_s / 1e9
    clocks = sampler.summary()

    # e2e: host buffers through gp_kmvm_host, copies inside the timed region
    e2e_steps = min(args.steps, 30)
    vh = torch.empty((nv, n), dtype=torch.float64).pin_memory()
    vh.copy_(V.cpu())
    oh = torch.empty_like(vh).pin_memory()
    lib = g.load_library()
    s = ctypes.c_void_p(stream.cuda_stream)
    for k in range(2):
        lib.gp_kmvm_host(plan._h, ctypes.c_void_p(vh[k].data_ptr()), 1,
                         ctypes.c_void_p(oh[k].data_ptr()), s)
    torch.cuda.synchronize()
    barrier(ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # (a) one call per MVM (copy in, apply, copy out, synchronise)
    e0.record(stream)
    for k in range(e2e_steps):
        st = lib.gp_kmvm_host(plan._h, ctypes.c_void_p(vh[k % nv].data_ptr()), 1,
                              ctypes.c_void_p(oh[k % nv].data_ptr()), s)
        assert st == 0
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    e2e_single_sec = max_over_ranks(e0.elapsed_time(e1) / 1e3, ws)
    # (b) one call for all the step's vectors (pinned buffers: the library pipelines the
    # host->device copy of column c+1, the apply of c and the device->host copy of c-1)
    lib.gp_kmvm_host(plan._h, ctypes.c_void_p(vh[0].data_ptr()), 3,
                     ctypes.c_void_p(oh[0].data_ptr()), s)
    torch.cuda.synchronize()
    barrier(ws)
    e0.record(stream)
    st = lib.gp_kmvm_host(plan._h, ctypes.c_void_p(vh[0].data_ptr()), e2e_steps,
                          ctypes.c_void_p(oh[0].data_ptr()), s)
    assert st == 0
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(ws)
    e2e_sec = max_over_ranks(e0.elapsed_time(e1) / 1e3, ws)
    e2e_value = sum_over_ranks(e2e_steps, ws) / e2e_sec

    line = {
        "metric": "kernel MVMs/sec (K.v, exact Matern ECDF decomposition) at N=1e6, d=1",
        "value": value,
        "unit": "MVM/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": sec_max / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE.json configs[1] recipe: x ~ N(0,1) seed 0, v ~ N(0,1))",
        "config": {
            "workload": "config2_d1_n1e6_nu52",
            "n": n, "d": 1, "nu": "5/2", "lengthscale": cfg.ell[0], "form": "L1(=product, d=1)",
            "setup": "once (sort + stored structure), outside the timed region",
            "l2": "inputs larger than L2: 100 distinct v and out buffers (1.6 GB) cycled",
            "launch": ("CUDA graph of K gp_kmvm calls (one cooperative kernel each), median of 5 replays"
                       if tinfo["graph"] else "gp_kmvm through ctypes, stream loop"),
            "stream_loop_ms_per_step": tinfo["stream_loop_ms_per_step"],
            "graph_replays": tinfo.get("replays", 1),
            "apply_ms_p10_p50_p90": [tinfo.get("apply_ms_p10"), tinfo.get("apply_ms_p50"),
                                     tinfo.get("apply_ms_p90")],
            "setup_s": tinfo["setup_s"],
            "parallelism": f"replicas x{ws}",
        },
        "gpu_launches": int(args.steps * launches),
        "clocks": clocks,
        "roofline": {
            "bound": "hbm", "kernel": d1_kernel_name(plan.query(7)),
            "achieved": achieved, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
            "frac": achieved / hbm,
            "traffic": ncu_traffic("d1_nu52_n1e6"),
            "algorithmic_bytes_per_launch": model_bytes,
            "launch_ms_mean": launch_s * 1e3,
            "launch_timing": ("graph replay of K launches / K" if tinfo["graph"]
                              else "per-launch CUDA events"),
            "launch_ms_isolated_mean": mean_l * 1e3, "launch_ms_isolated_median": med_l * 1e3,
        },
        "e2e": {"value": e2e_value, "unit": "MVM/s", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n, "steps": e2e_steps,
                "api": (f"gp_kmvm_host, {e2e_steps} pinned host vectors in one call (copies "
                        "pipelined with the applies, synchronised at the end)"),
                "per_call": {"value": sum_over_ranks(e2e_steps, ws) / e2e_single_sec,
                             "api": "gp_kmvm_host once per MVM (copy in, apply, copy out, sync)"}},
    }
    plan.close()

    extras = {}
    if not args.no_extras:
        # nu = 3/2 on the same config
        sx = min(args.steps, 1000)
        p3, _, smax3, s3, m3, _, _, t3 = measure(3, sx, 3)
        l3 = s3 / sx if t3["graph"] else m3
        extras["config2_d1_nu32"] = {"api": "gp_kmvm", "mvm_per_s": sum_over_ranks(sx, ws) / smax3,
                                     "launch_ms_mean": l3 * 1e3,
                                     "hbm_gbs": p3.model_bytes / l3 / 1e9,
                                     "frac_hbm": p3.model_bytes / l3 / 1e9 / hbm}
        p3.close()
        # the same apply in the plan's stored order (the operator inside CG: no gather/scatter)
        for nu2 in (5, 3):
            to_rank = lambda pl: torch.stack([pl.to_rank(V[i]) for i in range(nv)])
            pr, _, smr, sr, mr, _, _, tr = measure(nu2, sx, 3, vin=to_rank, rank_order=True)
            rb = n * 24   # t + v + out, all coalesced
            lr = sr / sx if tr["graph"] else mr   # per launch over the graph replay
            extras[f"config2_d1_nu{nu2}2_rank_order"] = {
                "api": "gp_kmvm_rank", "mvm_per_s": sum_over_ranks(sx, ws) / smr,
                "launch_ms_mean": lr * 1e3, "launch_ms_isolated_mean": mr * 1e3,
                "model_bytes": rb, "hbm_gbs": rb / lr / 1e9, "frac_hbm": rb / lr / 1e9 / hbm}
            pr.close()
        # f1: batched multi-RHS applies (one gp_kmvm call with nb fresh vectors)
        for nb, rank_order in ((16, False), (16, True)):
            pb = g.Plan(x, g.Kernel(5, cfg.ell), stream)
            VB = V[:nb] if not rank_order else torch.stack([pb.to_rank(V[i]) for i in range(nb)])
            OB = torch.empty_like(VB)
            lib = g.load_library()
            f = lib.gp_kmvm_rank if rank_order else lib.gp_kmvm
            vp, op, sp = ctypes.c_void_p(VB.data_ptr()), ctypes.c_void_p(OB.data_ptr()), ctypes.c_void_p(stream.cuda_stream)
            reps = 20
            for _ in range(3):
                f(pb._h, vp, nb, op, sp)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                f(pb._h, vp, nb, op, sp)
            e1.record(stream)
            torch.cuda.synchronize()
            sec = max_over_ranks(e0.elapsed_time(e1) / 1e3, ws)
            key = f"config2_d1_nu52_batched{nb}_{'rank' if rank_order else 'user'}_order"
            bpm = n * (24 if rank_order else 28)
            per = sec / (reps * nb)
            extras[key] = {"api": "gp_kmvm_rank" if rank_order else "gp_kmvm", "nrhs_per_call": nb,
                           "mvm_per_s": sum_over_ranks(reps * nb, ws) / sec,
                           "us_per_mvm": per * 1e6, "hbm_gbs": bpm / per / 1e9,
                           "frac_hbm": bpm / per / 1e9 / hbm}
            pb.close()
        extras["permutation_floor"] = permutation_floor(n, dev)
        extras.update(extra_configs(g, dev, stream, ws, rank, hbm, args))
    if extras:
        line["extra"] = extras
        rk = extras.get("config2_d1_nu52_rank_order")
        if rk:   # the CG operator: same kernel, vectors in the stored order (24 B/pt)
            line["roofline_rank_order"] = {
                "bound": "hbm", "kernel": d1_kernel_name(0, user=False), "achieved": rk["hbm_gbs"],
                "peak": hbm, "unit": "GB/s", "frac": rk["frac_hbm"],
                "algorithmic_bytes_per_launch": rk["model_bytes"], "launch_ms_mean": rk["launch_ms_mean"]}
        bt = extras.get("config2_d1_nu52_batched16_rank_order")
        if bt:
            line["roofline_batched16_rank_order"] = {
                "bound": "hbm", "achieved": bt["hbm_gbs"], "peak": hbm, "unit": "GB/s",
                "frac": bt["frac_hbm"], "us_per_mvm": bt["us_per_mvm"], "nrhs_per_call": 16}
        pf = extras.get("permutation_floor")
        if pf:
            line["user_order_floor"] = pf

    if rank == 0 and ws == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, two_nu, args.cpu_rows)
    return line


def permutation_floor(n, dev):
    """What the user-order permutations alone cost (profiles/r02_user_order_floor.md): a
    random gather v[p] and scatter o[p] = u of n doubles with PyTorch's own kernels (no
    arithmetic), back to back in one CUDA graph, against the 50 % budget of the whole
    apply (28 B/pt / (0.5 x peak))."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(7)
    p = torch.randperm(n, generator=g).to(dev)
    v = torch.randn(n, dtype=torch.float64, device=dev)
    o = torch.empty_like(v)
    u = torch.empty_like(v)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            torch.index_select(v, 0, p, out=u)
            o.index_copy_(0, p, u)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    R = 50
    with torch.cuda.graph(graph, stream=s):
        for _ in range(R):
            torch.index_select(v, 0, p, out=u)
            o.index_copy_(0, p, u)
    with torch.cuda.stream(s):
        graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        graph.replay()
        e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / R * 1e3
    hbm, _ = peaks()
    return {"gather_plus_scatter_us": us, "budget_50pct_us": 28 * n / (0.5 * hbm * 1e9) * 1e6,
            "how": "torch index_select + index_copy_ of 1e6 doubles through a random permutation, CUDA graph of 50",
            "evidence": "profiles/r02_user_order_floor.md (tools/micro/perm_floor.cu: 9.25 us L2-resident, ncu L2 requests)"}


def ncu_fp64(key):
    """FP64 FLOPs per apply of a workload (profiles/ncu_fp64.json, ncu instruction counts)
    and the derived FP64 peak (TFLOP/s), or (None, None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_fp64.json")) as f:
            d = json.load(f)
        return d.get(key), d.get("peak_fp64_tflops")
    except (OSError, ValueError):
        return None, None


def extra_configs(g, dev, stream, ws, rank, hbm, args):
    """d = 2 (config 3) and d = 3 (config 4) K.v; d=1,2,3 at N = 2^20 (the metric's
    'N=1e6, d=1..3'); config-5 CG solve time with --cg."""
    import torch
    out = {}

    def apply_stats(x_np, kern, reps, vecs=4, grad=False, fp64_key=None):
        x = torch.from_numpy(x_np).to(dev)
        t0 = time.perf_counter()
        plan = g.Plan(x, kern, stream)
        torch.cuda.synchronize()
        setup_s = time.perf_counter() - t0
        n = x_np.shape[0]
        V = torch.randn((vecs, n), dtype=torch.float64, device=dev)
        O = torch.empty_like(V)
        ap = Applier(g, plan, V, O, stream, grad=grad)
        # SURVEY §8(d) protocol: back-to-back applies in one CUDA graph (a stream loop of the
        # 6-7 launches of a d >= 2 apply is host-launch-bound below ~0.1 ms per apply)
        gr = None if args.no_graph else time_graph(
            lambda cs: Applier(g, plan, V, O, cs, grad=grad), reps, 3, ws, reps=3)
        timing = "CUDA graph of %d applies, median of 3 replays" % reps
        if gr is None:
            gr = time_applies(ap, reps, 3, stream, ws)
            timing = "stream loop of %d applies" % reps
        sec_max = gr[0]
        mean_l = sec_max / reps
        res = {"n": n, "setup_s": setup_s, "apply_ms": sec_max / reps * 1e3, "timing": timing,
               "mvm_per_s": sum_over_ranks(reps, ws) / sec_max,
               "launches_per_apply": plan.launches_per_apply,
               "model_bytes": plan.model_bytes,
               "model_gbs": plan.model_bytes / mean_l / 1e9,
               "frac_hbm": plan.model_bytes / mean_l / 1e9 / hbm,
               "struct_mb": plan.struct_bytes / 1e6}
        flop, peak = ncu_fp64(fp64_key) if fp64_key else (None, None)
        if flop:   # d >= 2 is bound by FP64 issue, not HBM: the ALU roofline
            tf = flop / (sec_max / reps) / 1e12
            res["alu_roofline"] = {"bound": "alu", "fp64_flop_per_apply": flop,
                                   "achieved": tf, "peak": peak, "unit": "TFLOP/s",
                                   "frac": tf / peak}
        plan.close()
        return res

    c3 = W.CONFIGS[3]
    out["config3_d2_n2e5_nu32_l1"] = apply_stats(W.config_points(c3), g.Kernel(3, c3.ell), 20,
                                                 fp64_key="config3_d2_nu32_l1")
    # config 3's rectangular product K_zx v (20,000 queries): union setup + applies
    x3 = torch.from_numpy(W.config_points(c3)).to(dev)
    z3 = torch.from_numpy(W.config_queries(c3)).to(dev)
    p3 = g.Plan(x3, g.Kernel(3, c3.ell), stream)
    v3 = torch.randn(c3.n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cr = p3.cross(z3, stream)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    o3 = cr.kzx(v3, stream=stream)
    torch.cuda.synchronize()
    gz = None if args.no_graph else time_graph(
        lambda cs: (lambda k: cr.kzx(v3, out=o3, stream=cs)), 10, 2, ws, reps=3)
    if gz is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(10):
            cr.kzx(v3, out=o3, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        gz = (e0.elapsed_time(e1) / 1e3, None)
    out["config3_kzx_m2e4"] = {"union_setup_s": t1 - t0, "apply_ms": gz[0] / 10 * 1e3,
                               "n": c3.n, "m": int(z3.shape[0])}
    cr.close()
    p3.close()
    out["config3_d2_n2e5_nu32_l1_dlengthscale"] = apply_stats(
        W.config_points(c3), g.Kernel(3, c3.ell), 20, grad=True)
    c2 = W.CONFIGS[2]
    out["config2_d1_n1e6_nu52_dlengthscale"] = apply_stats(
        W.config_points(c2), g.Kernel(5, c2.ell), 50, grad=True)
    c4 = W.CONFIGS[4]
    out["config4_d3_n5e5_nu52_l1"] = apply_stats(W.config_points(c4), g.Kernel(5, c4.ell), 5,
                                                 fp64_key="config4_d3_nu52_l1")
    for n1 in (1 << 20, 1 << 22):   # d = 1 above the single-chunk capacity (k_d1_coop)
        out[f"sweep_d1_n2^{n1.bit_length() - 1}_nu32"] = apply_stats(
            W.uniform_points(n1, 1, 1001), g.Kernel(3, (0.1,)), 50)
    for d, reps in [(2, 10), (3, 3)]:
        xn = W.uniform_points(1 << 20, d, 1000 + d)
        out[f"sweep_d{d}_n2^20_nu32_l1"] = apply_stats(xn, g.Kernel(3, (0.1,) * d), reps)
    # small n at d = 3 (the fused low kernels run in parts: 16 tiles fill the SMs) and the
    # d = 3 product form ((p+1)^2 re-weighted scan runs per level) on config 4's points
    out["sweep_d3_n2^14_nu32_l1"] = apply_stats(W.uniform_points(1 << 14, 3, 1014),
                                               g.Kernel(3, (0.1,) * 3), 20)
    out["config4_points_product_nu32"] = apply_stats(
        W.config_points(c4), g.Kernel(3, c4.ell, form=g.FORM_PRODUCT), 3)
    if not args.no_cg:
        c5 = W.CONFIGS[5]
        x = W.config_points(c5); y = W.config_response(c5, x)
        plan = g.Plan(torch.from_numpy(x).to(dev), g.Kernel(3, c5.ell, form=g.FORM_PRODUCT), stream)
        yt = torch.from_numpy(y).to(dev)
        torch.cuda.synchronize()
        cg_clock = ClockSampler(dev.index if dev.index is not None else 0)
        with cg_clock:   # a few seconds of sustained FP64 load: the SM clock is reported
            t0 = time.perf_counter()
            alpha, beta, info = plan.cg_solve(yt, c5.noise_sigma ** 2, mean=g.MEAN_AFFINE,
                                              rtol=1e-8, max_iter=40000)
            torch.cuda.synchronize()
            cg_s = time.perf_counter() - t0
        out["config5_cg"] = {"cg_solve_s": cg_s, "iters": info["iters"],
                             "relres_max": info["relres_max"], "rhs": 4, "beta": beta,
                             "ms_per_iter": cg_s / max(info["iters"], 1) * 1e3,
                             "preconditioner": "none (Alg 2 with s_P = I)",
                             "iteration": ("fused (apply epilogue q = Kp + s2 p with p.q partials, "
                                           "2 vector kernels), 8-iteration CUDA graphs"),
                             "clocks": cg_clock.summary()}
        # per-iteration split: the 4-column rank-order apply alone (CUDA graph of 20) vs
        # the whole iteration
        P4 = torch.randn((4, c5.n), dtype=torch.float64, device=dev)
        Q4 = torch.empty_like(P4)
        lib5 = g.load_library()
        cs5 = torch.cuda.Stream()
        def ap5(k, st=cs5):
            assert lib5.gp_kmvm_rank(plan._h, ctypes.c_void_p(P4.data_ptr()), 4,
                                     ctypes.c_void_p(Q4.data_ptr()), ctypes.c_void_p(st.cuda_stream)) == 0
        r5 = time_graph(lambda st: (lambda k: ap5(k, st)), 20, 3, 1, reps=3)
        # the same 4 columns through 400 CG iterations (all active: stopped by max_iter)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        try:
            plan.cg_solve(yt, c5.noise_sigma ** 2, mean=g.MEAN_AFFINE, rtol=1e-8, max_iter=400)
        except g.GPError:
            pass
        torch.cuda.synchronize()
        it4_ms = (time.perf_counter() - t0) / 400 * 1e3
        if r5:
            apply_ms = r5[0] / 20 * 1e3
            out["config5_cg"]["split_4_active_columns"] = {
                "iteration_ms": it4_ms, "apply_ms": apply_ms,
                "vector_ops_frac": max(0.0, (it4_ms - apply_ms) / it4_ms),
                "note": ("400 iterations with all 4 columns active (max_iter stop; includes "
                         "setup and the final true-residual apply) vs the 4-column rank-order "
                         "apply alone in a CUDA graph")}
        flop, peak = ncu_fp64("config5_d2_prod32_nrhs4")
        if flop:   # one 4-column apply per iteration dominates (vector updates are O(N))
            tf = flop * info["iters"] / cg_s / 1e12
            out["config5_cg"]["alu_roofline"] = {"bound": "alu", "fp64_flop_per_iter": flop,
                                                 "achieved": tf, "peak": peak,
                                                 "unit": "TFLOP/s", "frac": tf / peak}
        # the paper's preconditioned CG (App A: rank-k pivoted Cholesky + Woodbury), f3
        rank = 400
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pc = g.Precond(plan, rank, stream)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        alpha2, beta2, info2 = plan.cg_solve(yt, c5.noise_sigma ** 2, mean=g.MEAN_AFFINE,
                                             rtol=1e-8, max_iter=40000, precond=pc)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        out["config5_cg_precond"] = {"cg_solve_s": t2 - t1, "precond_setup_s": t1 - t0,
                                     "total_s": t2 - t0, "iters": info2["iters"],
                                     "relres_max": info2["relres_max"], "rhs": 4,
                                     "beta": beta2, "preconditioner": f"pivoted Cholesky rank {rank}",
                                     "ms_per_iter": (t2 - t1) / max(info2["iters"], 1) * 1e3}
        pc.close()
        # the setup again on the same plan: the first one includes the first-touch device
        # allocation of L (n x rank f64, 0.96 GB) through the caching allocator
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        pc = g.Precond(plan, rank, stream)
        torch.cuda.synchronize()
        out["config5_cg_precond"]["precond_setup_s_repeat"] = time.perf_counter() - t3
        pc.close()
        # posterior mean at the 10,000 queries (union setup + K_zx alpha + h(z)^T beta), the
        # first call (device allocations of the union structure included) and a repeat
        z5 = torch.from_numpy(W.config_queries(c5)).to(dev)
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            plan.predict(z5, alpha2, beta2, stream=stream)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        out["config5_predict"] = {"predict_s": ts[0], "predict_s_repeat": min(ts[1:]),
                                  "m": int(z5.shape[0]),
                                  "note": ("the first gp_predict builds the union x u z structure; "
                                           "repeats with the same z reuse it (bitwise check)")}
        pc.close()
        plan.close()
    return out


def cpu_baseline(cfg, two_nu, rows_n):
    import oracle
    x = W.config_points(cfg)
    v = W.config_vector(cfg, 0)
    rows = W.sample_rows(x, rows_n)
    nt = os.cpu_count() or 1
    oracle.kmvm_rows(x[:1000], v[:1000], two_nu, "l1", cfg.ell, rows=np.arange(10))  # load/warm
    t0 = time.perf_counter()
    oracle.kmvm_rows(x, v, two_nu, "l1", cfg.ell, rows=rows, nthreads=nt)
    dt = time.perf_counter() - t0
    full = dt * cfg.n / rows.size
    return {"value": 1.0 / full, "unit": "MVM/s", "cores": nt, "kind": "oracle",
            "sample": f"{rows.size} of {cfg.n} rows of one K.v (dense O(N) per row), "
                      f"{dt:.2f} s; full-MVM time extrapolated x{cfg.n / rows.size:.0f}",
            "seconds_per_mvm_extrapolated": full}


# ----------------------------------------------------------------------------- reference arm

def run_reference(args, ws, rank):
    import oracle
    if rank != 0:
        return None
    cfg = W.CONFIGS[2]
    x = W.config_points(cfg)
    nt = os.cpu_count() or 1
    # bound the whole run to a few minutes: rows per step from a short calibration
    oracle.kmvm_rows(x[:1000], np.ones(1000), 5, "l1", cfg.ell, rows=np.arange(10))
    t0 = time.perf_counter()
    oracle.kmvm_rows(x, W.config_vector(cfg, 0), 5, "l1", cfg.ell, rows=np.arange(64), nthreads=nt)
    per_row = (time.perf_counter() - t0) / 64
    budget = 120.0 / max(args.steps + args.warmup, 1)
    rows_per_step = int(max(16, min(1024, budget / per_row)))
    rng = np.random.default_rng(7)
    for k in range(args.warmup):
        oracle.kmvm_rows(x, W.config_vector(cfg, k), 5, "l1", cfg.ell,
                         rows=rng.choice(cfg.n, rows_per_step, replace=False), nthreads=nt)
    tot = 0.0
    for k in range(args.steps):
        rows = np.sort(rng.choice(cfg.n, rows_per_step, replace=False))
        v = W.config_vector(cfg, k)
        t0 = time.perf_counter()
        oracle.kmvm_rows(x, v, 5, "l1", cfg.ell, rows=rows, nthreads=nt)
        tot += time.perf_counter() - t0
    sec_per_mvm = tot / args.steps * cfg.n / rows_per_step
    value = 1.0 / sec_per_mvm
    sample = (f"{rows_per_step} random rows per step of the {cfg.n}-row K.v, "
              f"MVM time extrapolated x{cfg.n / rows_per_step:.0f}")
    return {
        "impl": "reference",
        "metric": "kernel MVMs/sec (K.v, exact Matern ECDF decomposition) at N=1e6, d=1",
        "value": value, "unit": "MVM/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec_per_mvm * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.json configs[1] recipe)",
        "config": {"workload": "config2_d1_n1e6_nu52", "n": cfg.n, "d": 1, "nu": "5/2",
                   "lengthscale": cfg.ell[0], "impl": "dense CPU oracle (oracle/), OpenMP"},
        "cpu_baseline": {"value": value, "unit": "MVM/s", "cores": nt, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "MVM/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cg", action="store_true", help="skip the config-5 CG solve")
    ap.add_argument("--no-graph", action="store_true", help="time a stream loop, not a graph")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=4096)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    ws, rank, local = dist_setup()
    if args.impl == "reference":
        line = run_reference(args, ws, rank)
    else:
        line = run_ours(args, ws, rank, local)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
