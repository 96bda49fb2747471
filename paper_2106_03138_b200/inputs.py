"""Seeded synthetic inputs for the five BASELINE.json configurations.

The recipes are SURVEY.md §8(d): numpy ``default_rng(seed)``, draws in the
listed order, Haar factors from the QR of a Gaussian matrix sign-fixed by
diag(R) (the reference's ``_haar_orthogonal``, harness.py:99-101).  Host
(numpy) generation is byte-reproducible and is what parity tests use; the two
large configs also have a device generator (torch, same recipe, different
random stream) for benchmarking, because a 16384^2 Haar QR on the host takes
minutes.  Which generator produced a number is recorded in bench output.
"""

from __future__ import annotations

import functools

import numpy as np


def _one_blas_thread(fn):
    """Host generators run with one BLAS thread: multi-threaded OpenBLAS QR/GEMM
    results depend on the thread count, and the inputs must be byte-reproducible."""
    @functools.wraps(fn)
    def wrapped(*a, **kw):
        try:
            from threadpoolctl import threadpool_limits
        except ImportError:  # pragma: no cover
            return fn(*a, **kw)
        with threadpool_limits(1):
            return fn(*a, **kw)
    return wrapped

CONFIGS = {
    "cfg1": dict(m=512, n=512, seed=0),
    "cfg2": dict(m=4096, n=4096, seed=1),
    "cfg3": dict(m=256, n=256, batch=1024, seed=3),
    "cfg4": dict(m=65536, n=1024, seed=4),
    "cfg5": dict(m=16384, n=16384, seed=4),
}


def nominal_flops(m: int, n: int) -> float:
    """The metric's flop count 2mn^2 - 2n^3/3 (BASELINE.json ``metric``)."""
    return 2.0 * m * n * n - 2.0 * n ** 3 / 3.0


def haar(rng: np.random.Generator, n: int) -> np.ndarray:
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    return q * np.sign(np.diagonal(r))


@_one_blas_thread
def cfg1(seed: int = 0, m: int = 512) -> np.ndarray:
    """512^2, sigma_i = 10^(-4(i-1)/383) for i <= 384, 1e-18 after (numerical rank 384)."""
    rng = np.random.default_rng(seed)
    U = haar(rng, m)
    V = haar(rng, m)
    i = np.arange(m)
    s = np.where(i < 384, 10.0 ** (-4.0 * i / 383.0), 1e-18)
    return np.asfortranarray((U * s) @ V.T)


@_one_blas_thread
def cfg2(seed: int = 1, n: int = 4096) -> np.ndarray:
    """n x n iid N(0,1)."""
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.standard_normal((n, n)))


@_one_blas_thread
def cfg3(seed: int = 3, batch: int = 1024, m: int = 256, r: int = 64) -> np.ndarray:
    """batch x (m x m): B (m x r) C (r x m) + 1e-10 E, draws B, C, E per matrix in order."""
    rng = np.random.default_rng(seed)
    out = np.empty((batch, m, m))
    for b in range(batch):
        B = rng.standard_normal((m, r))
        C = rng.standard_normal((r, m))
        E = rng.standard_normal((m, m))
        out[b] = B @ C + 1e-10 * E
    return out


@_one_blas_thread
def cfg4(seed: int = 4, m: int = 65536, n: int = 1024) -> np.ndarray:
    """U thin-orthonormal (sign-fixed QR of N(0,1) m x n), V Haar, sigma_i = i^-2,
    then column j scaled by 10^U(-6, 0)."""
    rng = np.random.default_rng(seed)
    q, r = np.linalg.qr(rng.standard_normal((m, n)))
    U = q * np.sign(np.diagonal(r))
    V = haar(rng, n)
    s = np.arange(1, n + 1, dtype=np.float64) ** -2.0
    A = (U * s) @ V.T
    A *= 10.0 ** rng.uniform(-6.0, 0.0, size=n)
    return np.asfortranarray(A)


@_one_blas_thread
def cfg5(seed: int = 4, n: int = 16384) -> np.ndarray:
    """Graded sigma_i = 10^(-30(i-1)/(n-1)), Haar U, V; then for j = 7 mod 8
    (0-based) A[:, j] = A[:, j-1] + 1e-12 N(0,1)."""
    rng = np.random.default_rng(seed)
    U = haar(rng, n)
    V = haar(rng, n)
    s = 10.0 ** (-30.0 * np.arange(n) / (n - 1))
    A = (U * s) @ V.T
    for j in range(7, n, 8):
        A[:, j] = A[:, j - 1] + 1e-12 * rng.standard_normal(n)
    return np.asfortranarray(A)


# ----------------------------------------------------------------------------
# device generators (same recipes, torch RNG) -- benchmark inputs only
# ----------------------------------------------------------------------------

def _torch_haar(n, gen, device):
    import torch
    g = torch.randn(n, n, generator=gen, dtype=torch.float64, device=device)
    q, r = torch.linalg.qr(g)
    return q * torch.sign(torch.diagonal(r))


def device_cfg(name: str, seed: int, device="cuda", n: int | None = None):
    """(n x lda)-shaped column-major device matrix for cfg2/cfg4/cfg5 (torch RNG)."""
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    if name == "cfg2":
        n = n or 4096
        return torch.randn(n, n, generator=gen, dtype=torch.float64, device=device).T
    if name == "cfg5":
        n = n or 16384
        U = _torch_haar(n, gen, device)
        V = _torch_haar(n, gen, device)
        s = 10.0 ** (-30.0 * torch.arange(n, dtype=torch.float64, device=device) / (n - 1))
        A = (U * s) @ V.T
        noise = torch.randn(n, n // 8, generator=gen, dtype=torch.float64, device=device)
        A[:, 7::8] = A[:, 6::8] + 1e-12 * noise
        return A
    if name == "cfg4":
        m, n = 65536, 1024
        q, r = torch.linalg.qr(torch.randn(m, n, generator=gen, dtype=torch.float64, device=device))
        U = q * torch.sign(torch.diagonal(r))
        V = _torch_haar(n, gen, device)
        s = torch.arange(1, n + 1, dtype=torch.float64, device=device) ** -2.0
        A = (U * s) @ V.T
        A *= 10.0 ** (torch.rand(n, generator=gen, dtype=torch.float64, device=device) * 6.0 - 6.0)
        return A
    raise ValueError(name)
