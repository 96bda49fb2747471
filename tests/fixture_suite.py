"""Restated generators for the reference's 40-matrix desk-scale fixture suite.

Test infrastructure: the reference commits 39 of these as MatrixMarket files
(pkg/fixtures/*.mtx) and rebuilds all 40 with ``harness.fixture_suite``
(harness.py:135-185).  The recipes below follow harness.py:83-132 (Kahan and
``random_rank_deficient``); ``tests/golden/golden_index.json`` stores the
sha256 of every input the reference produced, and ``test_oracle_golden.py``
checks these generators reproduce them byte for byte.
"""

from __future__ import annotations

import math

import numpy as np

EPS = float(np.finfo(np.float64).eps)


def kahan(n: int, theta: float) -> np.ndarray:
    """diag(s^i) * unit upper triangular with -cos(theta) above -- harness.py:83-96."""
    c, s = math.cos(theta), math.sin(theta)
    K = np.zeros((n, n), order="F")
    pw = s ** np.arange(n)
    for j in range(n):
        K[j, j] = pw[j]
        K[:j, j] = -c * pw[:j]
    return K


def _haar(rng, n):
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    return q * np.sign(np.diagonal(r))


def rank_deficient(m, n, r, gap, seed, kappa=1e3) -> np.ndarray:
    """U diag(s) V^T, r head values log-spaced in [1/kappa, 1], tail (1/kappa)/gap
    or eps/4 below 1e-10 -- harness.py:107-132."""
    rng = np.random.default_rng(seed)
    U = _haar(rng, m)
    V = _haar(rng, n)
    k = min(m, n)
    sv = np.zeros(k)
    if r > 0:
        sv[:r] = np.logspace(0.0, -math.log10(kappa), r)
        tail = (1.0 / kappa) / gap
        sv[r:] = tail if tail >= 1e-10 else EPS / 4.0
    return np.array((U[:, :k] * sv) @ V[:, :k].T, dtype=np.float64, order="F")


def suite():
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        return _suite()


def _suite():
    """(name, matrix) for all 40 members, in the reference's order -- harness.py:135-185."""
    out = []
    deficient = [
        (64, 48, 40), (64, 48, 24), (96, 64, 56), (96, 64, 32),
        (96, 96, 88), (96, 96, 64), (96, 96, 20), (128, 96, 90),
        (128, 96, 48), (128, 128, 120), (128, 128, 96), (160, 128, 112),
        (160, 128, 88), (192, 160, 150), (256, 192, 176), (60, 40, 15),
    ]
    for i, (m, n, r) in enumerate(deficient):
        out.append((f"rankdef_m{m}_n{n}_r{r}", rank_deficient(m, n, r, 1e9, seed=101 + i)))
    full = [
        (48, 48, 1e1), (64, 64, 1e2), (96, 72, 1e3), (96, 96, 1e4),
        (128, 96, 1e5), (128, 128, 1e6), (160, 160, 1e3), (80, 64, 1e2),
    ]
    for i, (m, n, kap) in enumerate(full):
        out.append((f"fullrank_m{m}_n{n}_k{kap:.0e}",
                    rank_deficient(m, n, min(m, n), 1e1, seed=151 + i, kappa=kap)))
    cliffs = [
        (64, 48, 32, 1e4, 1e3), (96, 64, 48, 1e4, 1e3), (96, 96, 80, 1e5, 1e2),
        (128, 96, 80, 1e4, 1e3), (128, 128, 112, 1e4, 1e2), (96, 96, 72, 1e4, 1e3),
        (160, 128, 116, 1e4, 1e3), (72, 72, 48, 1e4, 1e3),
    ]
    for i, (m, n, r, gap, kap) in enumerate(cliffs):
        out.append((f"cliff_m{m}_n{n}_r{r}_g{gap:.0e}",
                    rank_deficient(m, n, r, gap, seed=201 + i, kappa=kap)))
    for n, c in [(64, 0.05), (96, 0.02), (96, 0.05), (128, 0.01)]:
        out.append((f"kahan_n{n}_c{c:.2f}", kahan(n, math.acos(c))))
    extras = [(192, 48, 36, 1e9, 1e3), (48, 96, 40, 1e9, 1e3), (96, 96, 94, 1e9, 1e3)]
    for i, (m, n, r, gap, kap) in enumerate(extras):
        out.append((f"rankdef_m{m}_n{n}_r{r}", rank_deficient(m, n, r, gap, seed=251 + i, kappa=kap)))
    out.append(("fullrank_m128_n128_k1e+07",
                rank_deficient(128, 128, 128, 1e1, seed=260, kappa=1e7)))
    return out
