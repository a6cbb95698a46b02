"""World-size-2 (gloo, CPU) check of bench.py's multi-rank host logic: each
rank draws its own seeded rows (weak scaling, no data-path collective) and the
reported step time is the max over ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    g = bench.make_inputs(1, rank)
    digest = float(np.abs(g).sum())
    mx = bench.max_over_ranks(1.5 + rank, dist, "cpu")
    gathered = [None] * world
    dist.all_gather_object(gathered, digest)
    q.put((rank, mx, gathered))
    dist.destroy_process_group()


def test_two_ranks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, gathered in res:
        assert mx == pytest.approx(2.5)            # max over ranks
        assert gathered[0] != gathered[1]          # each rank owns distinct rows


def test_bench_launcher_two_ranks():
    """`python bench.py --gpus 2` relaunches itself under torch.distributed.run (one process
    per GPU); the dry run exercises that launcher, the rendezvous on 127.0.0.1, per-rank
    seeded inputs and the max-over-ranks step time on gloo, and rank 0 alone prints one line."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run-gloo"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["ms_per_step"] == pytest.approx(2.0) and d["distinct_inputs"]
