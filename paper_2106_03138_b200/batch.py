"""Batches of independent matrices (BASELINE cfg3) and their multi-GPU sharding.

A single matrix does not shard: the QRDM panel recursion is sequential
(SURVEY §8e), so one matrix always runs on one GPU.  A batch of independent
matrices is partitioned evenly over the ranks of a torch.distributed job; each
rank factors its contiguous slice through ``dmqr_qrdm_batched_f64`` and the
small per-matrix outputs (rank, n_factored, stopped_early, steps, permutation,
coefficients) are gathered with ``all_gather_into_tensor`` -- NCCL on GPUs --
which is the only collective (north_star: "NCCL is used only to gather
results").  The packed factors stay on the rank that computed them unless
asked for.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .rrqr import (
    DMParams,
    Permutation,
    RRQRResult,
    StopCriterion,
    rule_code,
    _check,
    _steps_from_raw,
    _torch,
    engine_k_dm,
    lda_for,
    replay_counters,
    swap_capacity,
)


def shard(batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of a batch owned by ``rank`` (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return batch * rank // world, batch * (rank + 1) // world


@dataclass
class BatchFactor:
    """Device outputs of a batched factorization (matrices [lo, hi) of the full batch)."""

    buf: object        # torch (b, n, lda) column-major packed factors
    m: int
    n: int
    lda: int
    coeffs: object     # torch (b, kmax)
    perm: object       # torch int64 (b, n)
    swaps: object      # torch int64 (b, swap_cap, 2)
    steps: object      # torch uint8 (b, step_cap * STEP_BYTES)
    infos: list        # host dmqr_info per matrix
    step_cap: int
    swap_cap: int

    @property
    def ranks(self) -> np.ndarray:
        return np.array([int(i.rank) for i in self.infos], dtype=np.int64)

    def result(self, i: int) -> RRQRResult:
        """RRQRResult of matrix i (host copies), identical in form to qrdm2's."""
        info = self.infos[i]
        steps = _steps_from_raw(self.steps[i].cpu().numpy(), int(info.n_steps))
        p = Permutation(self.n)
        p.forward = self.perm[i].cpu().numpy().astype(np.intp)
        p.swaps = [(int(a), int(b)) for a, b in self.swaps[i, : int(info.n_swaps)].cpu().numpy()]
        packed = self.buf[i, : self.n, : self.m].T.cpu().numpy()
        return RRQRResult(packed=np.asfortranarray(packed), coeffs=self.coeffs[i].cpu().numpy(), perm=p,
                          rank=int(info.rank), step_log=steps, n_factored=int(info.n_factored),
                          stopped_early=bool(info.stopped_early), counters=replay_counters(self.m, self.n, steps))


def to_batch_work(A, device=None):
    """(b, n, lda) column-major float64 device copy of a (b, m, n) batch."""
    torch = _torch()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    t = A if isinstance(A, torch.Tensor) else torch.as_tensor(np.asarray(A, dtype=np.float64))
    if t.dim() != 3:
        raise ValueError(f"expected a (batch, m, n) array, got ndim={t.dim()}")
    t = t.to(device=dev, dtype=torch.float64)
    b, m, n = (int(x) for x in t.shape)
    lda = lda_for(m)
    buf = torch.zeros((b, max(n, 1), lda), dtype=torch.float64, device=dev)
    if b and m and n:
        buf[:, :n, :m].copy_(t.transpose(1, 2))
    return buf, m, n, lda


def factorize_batch(A, params: DMParams = DMParams(), stop: StopCriterion = StopCriterion(),
                    break_check: bool = True, lanes: int = 16, work=None) -> BatchFactor:
    """QRDM2 (break_check) / QRDM of every matrix of a (b, m, n) batch on the current GPU."""
    torch = _torch()
    lib = _lib.load()
    buf, m, n, lda = work if work is not None else to_batch_work(A)
    b = int(buf.shape[0])
    dev = buf.device
    kmax = min(m, n)
    step_cap = max(kmax, 1)
    k_dm = engine_k_dm(params.k_dm, n)
    swap_cap = swap_capacity(kmax, k_dm)
    p = _lib.Params(tau=float(params.tau), delta=float(params.delta), epsilon=float(stop.epsilon),
                    k_dm=k_dm, use_delta_max=int(bool(params.use_delta_max)),
                    stop_rule=rule_code(stop), break_check=int(bool(break_check)), trace_norms=0,
                    max_steps=0)
    coeffs = torch.zeros((b, max(kmax, 1)), dtype=torch.float64, device=dev)
    perm = torch.zeros((b, max(n, 1)), dtype=torch.int64, device=dev)
    swaps = torch.empty((b, swap_cap, 2), dtype=torch.int64, device=dev)
    steps = torch.empty((b, step_cap * _lib.STEP_BYTES), dtype=torch.uint8, device=dev)
    infos = (_lib.Info * max(b, 1))()
    group = max(1, int(lib.dmqr_batched_group(m, n)))  # matrices per lane launch (grid.z)
    lanes = max(1, min(int(lanes), max(b, 1), -(-max(b, 1) // group)))
    wsb = int(lib.dmqr_batched_workspace_bytes(m, n, C.byref(p), lanes))
    ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=dev)
    sh = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    stride = int(buf.shape[1]) * lda
    _check(lib.dmqr_qrdm_batched_f64(buf.data_ptr(), b, m, n, lda, stride, C.byref(p), coeffs.data_ptr(),
                                     perm.data_ptr(), swaps.data_ptr(), swap_cap, steps.data_ptr(), step_cap,
                                     infos, lanes, ws.data_ptr(), wsb, sh))
    return BatchFactor(buf, m, n, lda, coeffs[:, :kmax], perm[:, :n], swaps, steps, list(infos)[:b], step_cap,
                       swap_cap)


def qrdm2_batched(A, params: DMParams = DMParams(), stop: StopCriterion = StopCriterion(), lanes: int = 16):
    """List of RRQRResult, one per matrix of the (b, m, n) batch."""
    f = factorize_batch(A, params, stop, True, lanes)
    return [f.result(i) for i in range(len(f.infos))]


def summary_tensor(f: BatchFactor, device):
    """(b, 4 + n + kmax) float64 summary rows: rank, n_factored, stopped, n_steps, perm, coeffs.
    (Host-side table logic: plain torch, any device.)"""
    import torch
    b = len(f.infos)
    rows = [[i.rank, i.n_factored, i.stopped_early, i.n_steps] for i in f.infos]
    head = torch.tensor(rows, dtype=torch.float64, device=device).reshape(b, 4)
    return torch.cat([head, f.perm.to(torch.float64), f.coeffs], dim=1)


def gather_summaries(local, batch: int, group=None):
    """all_gather the per-rank summary rows into the full (batch, width) table, in batch order.

    Ranks own contiguous slices whose sizes differ by at most one; every rank pads
    to the largest slice so ``all_gather_into_tensor`` sees equal shapes.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    width = int(local.shape[1])
    per = -(-batch // world)
    pad = torch.zeros((per, width), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * per, width), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    rows = []
    for r in range(world):
        lo, hi = shard(batch, r, world)
        rows.append(out[r * per: r * per + (hi - lo)])
    return torch.cat(rows, dim=0)
