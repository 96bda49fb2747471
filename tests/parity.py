"""Parity checks of a GPU result against the CPU oracle (margin-aware).

The north star asks for identical permutation and rank wherever selection
margins exceed 1e3*eps, |diag R| within 1e-10 relative on the revealed part,
and residual / orthogonality <= 50 n eps.  Margins come from the oracle's
decision trace; each margin is scaled by the amplification a_max0/u_max of the
step it was taken in, because trailing quantities carry absolute error
~eps*||A||.
"""

from __future__ import annotations

import numpy as np

from oracle import qrdm_oracle as O

EPS = O.EPS
MARGIN = 1e3 * EPS


def robust_prefix(ref: O.OracleResult):
    """Columns [0, cut) whose pivots were decided with margin > 1e3 eps (amplified),
    and whether the whole run (incl. rank/stop) was robust.  SURVEY §8d: identical
    permutation up to the first ambiguous decision."""
    fa = ref.margins.get("first_ambiguous")
    if fa is None:
        return ref.n_factored, True
    return int(fa), False


def diag_close(d_gpu, d_ref, n) -> tuple[bool, float]:
    """| |d_gpu| - |d_ref| | <= 1e-10 |d_ref| + n eps |d_1|."""
    if hasattr(d_gpu, "cpu"):  # a device result (torch)
        d_gpu = d_gpu.cpu().numpy()
    a, b = np.abs(np.asarray(d_gpu)), np.abs(np.asarray(d_ref))
    k = min(a.size, b.size)
    if k == 0:
        return True, 0.0
    err = np.abs(a[:k] - b[:k])
    tol = 1e-10 * b[:k] + n * EPS * b[0]
    worst = float(np.max(err / np.maximum(tol, 1e-300)))
    return bool(np.all(err <= tol)), worst


def residuals(A, res, Q=None):
    """(||A P - Q R||_F / ||A||_F, ||Q^T Q - I||_F) using the device-formed Q."""
    from paper_2106_03138_b200 import reconstruct

    A = np.asarray(A, dtype=np.float64)
    if Q is None:
        Q, R = reconstruct(res)
    else:
        _, R = reconstruct(res)
    nA = max(np.linalg.norm(A), np.finfo(float).tiny)
    resid = np.linalg.norm(A[:, res.perm.forward] - Q @ R) / nA
    orth = np.linalg.norm(Q.T @ Q - np.eye(Q.shape[1]))
    return float(resid), float(orth)
