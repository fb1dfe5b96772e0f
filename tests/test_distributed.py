"""Multi-process plumbing of bench.py / the one-process-per-GPU layout, on CPU with gloo
(world size 2): shard ranges, the NCCL-id broadcast, max-over-ranks timing, and the reference
arm under torchrun (rank 0 alone prints)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as tdist
    from paper_2602_03609_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = D.broadcast_object(bytes(range(128)) if rank == 0 else None)
        mx = D.max_over_ranks(1.5 + rank)
        sm = D.sum_over_ranks(1.0 + rank)
        q.put((rank, uid, mx, sm, D.shard_range(1_100_000, rank, world)))
    finally:
        tdist.destroy_process_group()


def test_shard_ranges_partition():
    from paper_2602_03609_b200 import dist as D
    for n in (0, 1, 7, 1000, 1_100_000):
        for world in (1, 2, 3, 4, 8):
            r = [D.shard_range(n, k, world) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(r[k][1] == r[k + 1][0] for k in range(world - 1))
            # the engine's split: static_cast<long long>(n) * rank / world
            assert all(lo == n * k // world for k, (lo, _) in enumerate(r))


def test_gloo_world2_collectives():
    import torch.multiprocessing as mp
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[0] for r in res] == [0, 1]
    assert all(r[1] == bytes(range(128)) for r in res)  # NCCL unique id reaches every rank
    assert all(r[2] == 2.5 for r in res)                # max over ranks
    assert all(r[3] == 3.0 for r in res)
    assert res[0][4] == (0, 550_000) and res[1][4] == (550_000, 1_100_000)


def test_reference_arm_under_torchrun():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1", "--workload", "vecchia",
           "--stations", "60", "--days", "5"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"
