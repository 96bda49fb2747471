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

from paper_2106_03138_b200.batch import gather_summaries, shard


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
