"""Multi-rank (N>1) host path on CPU: gloo, world_size 2.

The row-shard partition and the final gather are exercised with a stand-in
compute function — the CPU oracle, used here strictly as the checker/stand-in
for the per-rank GPU forward — and must reproduce the single-process result
bit for bit (rows are independent)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_19689_b200.sharding import shard_bounds, run_sharded
from paper_2510_19689_b200 import workloads as W


def test_shard_bounds_partition():
    for rows in (0, 1, 7, 128, 1000, 65536):
        for world in (1, 2, 3, 4, 8):
            b = shard_bounds(rows, world)
            assert b[0][0] == 0 and b[-1][1] == rows
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, rows, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import tabnet_oracle as O
        m = W.make_model("adult")
        x = W.make_inputs(W.WORKLOADS["adult"], rows).astype(np.float64)

        def forward(xs):
            r = O.apply_model(m, xs)
            return {k: torch.from_numpy(r[k]) for k in ("logits", "probabilities", "masks", "importance")}

        full = run_sharded(forward, x, rank, world)
        # timing reduction used by bench.py: max over ranks
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            q.put(({k: v.numpy() for k, v in full.items()}, float(t.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rows", [257, 1000])
def test_gloo_world2_shard_gather_bitwise(rows):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, rows, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import tabnet_oracle as O
    m = W.make_model("adult")
    x = W.make_inputs(W.WORKLOADS["adult"], rows).astype(np.float64)
    ref = O.apply_model(m, x)
    for k in ("logits", "probabilities", "masks", "importance"):
        assert np.array_equal(full[k], ref[k]), k
    assert tmax == 2.0
