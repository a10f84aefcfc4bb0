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
