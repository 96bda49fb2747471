"""World-size-2 gloo tests (CPU) for the batched multi-GPU path: even sharding
of a batch of independent matrices and the all_gather of per-matrix results
back into batch order.  The GPU factorization itself is exercised by -m gpu
tests; here each rank contributes rows derived from the global matrix index."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2106_03138_b200.batch import gather_summaries, shard, summary_tensor


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, batch, width, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard(batch, rank, world)
        # stand-in for summary_tensor(): row i = global matrix index, then a rank tag
        local = torch.stack([torch.full((width,), float(i)) for i in range(lo, hi)]) if hi > lo else \
            torch.zeros((0, width))
        if hi > lo:
            local[:, 1] = float(rank)
        full = gather_summaries(local, batch)
        q.put((rank, full.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [7, 8, 1024])
def test_gloo_world2_shard_and_gather(batch):
    world, width = 2, 5
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, batch, width, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        full = torch.tensor(out[r])
        assert full.shape == (batch, width)
        assert torch.equal(full[:, 0], torch.arange(batch, dtype=full.dtype))  # batch order
        owner = torch.tensor([0.0 if i < shard(batch, 1, world)[0] else 1.0 for i in range(batch)])
        assert torch.equal(full[:, 1], owner)


def _summary_worker(rank, world, port, batch, q):
    """Each rank builds the per-matrix summary rows of its slice with the real
    summary_tensor (rank, n_factored, stopped, n_steps, perm, coeffs) from a
    stand-in BatchFactor, then gathers them: the table bench.py gathers inside
    the timed cfg3 region."""
    from types import SimpleNamespace

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard(batch, rank, world)
        m = n = 6
        infos = [SimpleNamespace(rank=n - (i % 2), n_factored=n, stopped_early=i % 2, n_steps=2 + i % 3)
                 for i in range(lo, hi)]
        perm = torch.stack([torch.roll(torch.arange(n), i) for i in range(lo, hi)]) if hi > lo else \
            torch.zeros((0, n), dtype=torch.int64)
        coeffs = torch.stack([torch.full((min(m, n),), i / 10.0) for i in range(lo, hi)]) if hi > lo else \
            torch.zeros((0, min(m, n)))
        f = SimpleNamespace(infos=infos, perm=perm, coeffs=coeffs.double())
        local = summary_tensor(f, torch.device("cpu"))
        assert local.shape == (hi - lo, 4 + n + min(m, n))
        q.put((rank, gather_summaries(local, batch).tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [5, 1024])
def test_gloo_world2_summary_tensor_gather(batch):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_summary_worker, args=(r, world, port, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        full = torch.tensor(out[r], dtype=torch.float64)
        assert full.shape == (batch, 4 + 6 + 6)
        i = torch.arange(batch, dtype=torch.float64)
        assert torch.equal(full[:, 0], 6 - (i % 2))                      # rank column, batch order
        assert torch.equal(full[:, 3], 2 + i % 3)                        # n_steps
        assert torch.equal(full[:, 4], (-i) % 6)                         # perm[0] of roll(arange, i)
        assert torch.allclose(full[:, -1], i / 10.0)                     # coeffs


def test_shard_partition():
    for batch in (0, 1, 7, 1024):
        for world in (1, 2, 4, 8):
            spans = [shard(batch, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(8, 2, 2)
