"""Host-side multi-rank logic of bench.py (replicas, max/sum over ranks) on CPU with gloo,
world size 2 (the path runs as independent replicas, no data-path collective)."""
import os
import socket
import subprocess
import sys
import textwrap

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


WORKER = textwrap.dedent("""
    import os, sys, json
    sys.path.insert(0, {root!r})
    import bench
    ws, rank, local = bench.dist_setup()
    assert ws == 2
    import torch.distributed as dist
    assert dist.get_backend() == "gloo"
    # each replica reports its own time / work; the job takes the max time, summed work
    t = 1.0 + rank            # rank 1 is the slower replica
    mx = bench.max_over_ranks(t, ws)
    sm = bench.sum_over_ranks(100.0, ws)
    bench.barrier(ws)
    print(json.dumps({{"rank": rank, "max": mx, "sum": sm}}), flush=True)
    dist.destroy_process_group()
""")


def test_replica_reductions_gloo_ws2(tmp_path):
    script = tmp_path / "w.py"
    script.write_text(WORKER.format(root=ROOT))
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE="2",
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=180) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
    import json
    res = [json.loads(o.strip().splitlines()[-1]) for o, _ in outs]
    for r in res:
        assert r["max"] == 2.0 and r["sum"] == 200.0


def test_reference_arm_other_ranks_exit_without_work():
    """Under torchrun only rank 0 runs the CPU reference arm (bench.run_reference)."""
    sys.path.insert(0, ROOT)
    import bench

    class A:
        steps, warmup = 1, 0
    assert bench.run_reference(A(), 2, 1) is None


SHARD_WORKER = textwrap.dedent("""
    import os, sys, json
    sys.path.insert(0, {root!r})
    import numpy as np, torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    rank, ws = dist.get_rank(), dist.get_world_size()
    import paper_2508_01864_b200 as g
    import oracle
    res = {{}}
    # (1) the work split of gp_kmvm_partial (host-only C ABI): disjoint, covering
    for n, d in [(5000, 3), (200000, 2), (500000, 3), (1, 2), (2049, 3)]:
        mine = g.shard_ranges(n, d, rank, ws)
        allr = [None] * ws
        dist.all_gather_object(allr, mine)
        res[f"{{n}}_{{d}}"] = allr
    # (2) the collective of the sharded apply: per-rank partial products summed by one
    # all-reduce equal the whole product (partials here: the oracle's K v over this rank's
    # share of the sources -- the same sum-of-partials identity the GPU shards rely on)
    rng = np.random.default_rng(3)
    x = rng.random((300, 3)); v = rng.standard_normal(300)
    src = np.zeros(300); src[rank::ws] = v[rank::ws]
    part = torch.from_numpy(oracle.kmvm_rows(x, src, 5, "l1", (0.2, 0.3, 0.5), 1.0))
    dist.all_reduce(part, op=dist.ReduceOp.SUM)
    full = oracle.kmvm_rows(x, v, 5, "l1", (0.2, 0.3, 0.5), 1.0)
    res["allreduce_err"] = float(np.max(np.abs(part.numpy() - full)))
    res["scale"] = float(np.max(np.abs(full)))
    print(json.dumps(res), flush=True)
    dist.destroy_process_group()
""")


def test_sharded_apply_split_and_collective_gloo_ws2(tmp_path):
    """gp_kmvm_partial's work split (gp_shard_ranges, host-only) and the all-reduce of the
    shards' partial products, world size 2 on gloo (the GPU shards themselves are checked
    against the whole apply in tests/test_gpu_parity.py::test_sharded_apply_sums_to_kv)."""
    script = tmp_path / "s.py"
    script.write_text(SHARD_WORKER.format(root=ROOT))
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE="2",
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=300) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
    import json
    res = [json.loads(o.strip().splitlines()[-1]) for o, _ in outs]
    for key in ("5000_3", "200000_2", "500000_3", "1_2", "2049_3"):
        n = int(key.split("_")[0])
        tiles = (n + 1023) // 1024
        (t0, t1), (i0, i1) = res[0][key][0]
        (u0, u1), (j0, j1) = res[0][key][1]
        assert res[0][key] == res[1][key]               # every rank derives the same split
        assert t0 == 0 and t1 == u0 and u1 == tiles      # tiles: disjoint and covering
        assert i0 == 0 and i1 == j0 and j1 >= j0         # carried-pass items likewise
        assert abs((t1 - t0) - (u1 - u0)) <= 1           # balanced
    for r in res:
        assert r["allreduce_err"] <= 1e-12 * r["scale"]
