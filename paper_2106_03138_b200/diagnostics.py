"""Rank-revealing diagnostics of a factorization.

* ``jacobi_svd`` / ``jacobi_svd_batched``: singular values by one-sided Jacobi
  on the device (``dmqr_jacobi_svd_batched_f64``, csrc/jacobi.cuh) -- the
  counterpart of the reference's verification oracle ``jacobi_svd``
  (svd.py:117-143): the same rotation and stopping rule, the same 512-column
  desk-scale cap and wide-matrix transpose, ``numerical_rank`` =
  #{sigma_i > eps n sigma_1} (svd.py:57, 139).  One CTA per matrix, so a whole
  batch (BASELINE cfg3: 1024 x 256^2) runs in one launch.
* ``ratio_fields``: harness._ratio_fields (harness.py:201-216) for one result:
  the sorted |diag R| over the numerical rank against the singular values
  (rd) and the singular values of R11 against them (rs), given the input's
  spectrum; sigma(R11) by the device Jacobi SVD.
* ``ratio_fields_batched``: the same for a whole batch (BatchFactor or a list of
  results), every SVD on the device in two batched launches.

Verification tooling, off the factorization path.  Like the product API, it
raises without a CUDA device (no CPU fallback).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

EPS = float(np.finfo(np.float64).eps)
MAX_COLS = 512  # svd.py: _MAX_COLS


@dataclass
class SpectrumReport:
    """svd.SpectrumReport (svd.py:54-58)."""

    sigmas: np.ndarray  # descending
    numerical_rank: int
    convergence_sweeps: int
    converged: bool = True


def jacobi_svd_batched(X, tol: float = 1e-15, max_sweeps: int = 30) -> list[SpectrumReport]:
    """Spectra of a (b, m, n) batch (numpy or torch) by device one-sided Jacobi."""
    from . import _lib
    from .rrqr import _check, _torch

    torch = _torch()
    t = X if isinstance(X, torch.Tensor) else torch.as_tensor(np.asarray(X, dtype=np.float64))
    if t.dim() != 3:
        raise ValueError("oracle input must be a (batch, m, n) array")
    b, m, n_cols = (int(x) for x in t.shape)
    if m < n_cols:  # wide: the spectrum of the transpose (svd.py:131)
        t = t.transpose(1, 2)
        m, n = n_cols, m
    else:
        n = n_cols
    if n > MAX_COLS:
        raise ValueError(f"oracle guard: {n} columns exceeds the desk-scale cap {MAX_COLS}")
    dev = torch.device("cuda", torch.cuda.current_device())
    work = torch.empty((b, n, m), dtype=torch.float64, device=dev)  # column-major copies
    work.copy_(t.to(device=dev, dtype=torch.float64).transpose(1, 2))
    sig = torch.zeros((b, max(n, 1)), dtype=torch.float64, device=dev)
    sweeps = torch.zeros(max(b, 1), dtype=torch.int32, device=dev)
    conv = torch.ones(max(b, 1), dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev)
    _check(_lib.load().dmqr_jacobi_svd_batched_f64(work.data_ptr(), b, m, n, max(m, 1), max(m, 1) * max(n, 1),
                                                   float(tol), int(max_sweeps), sig.data_ptr(), sweeps.data_ptr(),
                                                   conv.data_ptr(), C.c_void_p(st.cuda_stream)))
    s = torch.sort(sig[:, :n], dim=1, descending=True).values.cpu().numpy()
    sw, cv = sweeps.cpu().numpy(), conv.cpu().numpy()
    out = []
    for i in range(b):
        s0 = s[i, 0] if n else 0.0
        rank = int(np.count_nonzero(s[i] > EPS * n_cols * s0))
        out.append(SpectrumReport(s[i].copy(), rank, int(sw[i]), bool(cv[i])))
    return out


def jacobi_svd(A, tol: float = 1e-15, max_sweeps: int = 30) -> SpectrumReport:
    """svd.jacobi_svd (svd.py:117-143) on the device, one matrix."""
    A = A if not isinstance(A, np.ndarray) else np.asarray(A, dtype=np.float64)
    if getattr(A, "ndim", None) != 2:
        raise ValueError("oracle input must be 2-d")
    return jacobi_svd_batched(A[None], tol, max_sweeps)[0]


def _rdiag(result, packed) -> np.ndarray:
    """|diag R| over the factored columns (RRQRResult.r_diagonal, rrqr.py:156-158)."""
    return np.abs(np.diagonal(packed)[: int(result.n_factored)])


def _fields(d_sorted: np.ndarray, sigma: np.ndarray, sig_r11: np.ndarray, k: int, flags: str):
    if k == 0:
        return 1.0, 1.0, 1.0, 1.0, flags
    rd = d_sorted[:k] / sigma[:k]
    rs = sig_r11[:k] / sigma[:k]
    return float(rd.min()), float(rd.max()), float(rs.min()), float(rs.max()), flags


def ratio_fields(result, sigmas, n_r: int, r11_svd: str = "device") -> tuple[float, float, float, float, str]:
    """(ratio_d_min, ratio_d_max, ratio_s_min, ratio_s_max, flags) as harness._ratio_fields,
    given the input's spectrum (``sigmas`` descending, numerical rank ``n_r``).
    sigma(R11) by the device Jacobi SVD, or ``r11_svd="host"`` (LAPACK) for
    host-only checks of the bookkeeping."""
    packed = result.packed if isinstance(result.packed, np.ndarray) else result.packed.cpu().numpy()
    flags = ""
    k = min(int(n_r), int(result.n_factored))
    if k < n_r:
        flags = "short_factorization"
    if k == 0:
        return 1.0, 1.0, 1.0, 1.0, flags
    sigma = np.asarray(sigmas, dtype=np.float64)
    d = np.sort(_rdiag(result, packed)[:n_r])[::-1]
    r11 = np.triu(packed[:k, :k])
    sig_r11 = np.linalg.svd(r11, compute_uv=False) if r11_svd == "host" else jacobi_svd(r11).sigmas
    return _fields(d, sigma, sig_r11, k, flags)


def ratio_fields_batched(results, A_batch, rank_eps1: float | None = None):
    """harness._ratio_fields for every matrix of a batch, with both SVDs on the
    device: the spectra of the inputs (n_r = their numerical rank, or
    #{sigma > rank_eps1 sigma_1} as compare_run's ``rank_eps1``, harness.py:244-247)
    and of the R11 blocks (zero-padded to a common size; the padding adds zero
    singular values only).  ``results``: a BatchFactor or a list of RRQRResult.
    Returns (list of 5-tuples, list of SpectrumReport of the inputs)."""
    if hasattr(results, "result") and hasattr(results, "infos"):
        results = [results.result(i) for i in range(len(results.infos))]
    specs = jacobi_svd_batched(A_batch)
    b = len(results)
    if b == 0:
        return [], specs
    ks, nrs, flags = [], [], []
    for res, sp in zip(results, specs):
        n_r = (int(np.count_nonzero(sp.sigmas > rank_eps1 * sp.sigmas[0])) if rank_eps1 is not None
               else sp.numerical_rank)
        k = min(n_r, int(res.n_factored))
        nrs.append(n_r)
        ks.append(k)
        flags.append("short_factorization" if k < n_r else "")
    kmax = max(max(ks), 1)
    r11 = np.zeros((b, kmax, kmax))
    for i, res in enumerate(results):
        k = ks[i]
        packed = res.packed if isinstance(res.packed, np.ndarray) else res.packed.cpu().numpy()
        r11[i, :k, :k] = np.triu(packed[:k, :k])
    sr = jacobi_svd_batched(r11)
    out = []
    for i, res in enumerate(results):
        packed = res.packed if isinstance(res.packed, np.ndarray) else res.packed.cpu().numpy()
        d = np.sort(_rdiag(res, packed)[:nrs[i]])[::-1]
        out.append(_fields(d, specs[i].sigmas, sr[i].sigmas, ks[i], flags[i]))
    return out, specs
