"""Rank-revealing diagnostics of a factorization (host side).

``ratio_fields`` mirrors harness._ratio_fields (harness.py:201-216): the sorted
|diag R| over the numerical rank against the singular values (rd), and the
singular values of R11 against them (rs).  The reference computes the
singular values with its own one-sided Jacobi SVD (svd.py); here the caller
passes them in (known by construction for the BASELINE spectra, or from any
SVD), and sigma(R11) comes from LAPACK on the host -- verification tooling, off
the factorization path.
"""

from __future__ import annotations

import numpy as np


def ratio_fields(result, sigmas, n_r: int) -> tuple[float, float, float, float, str]:
    """(ratio_d_min, ratio_d_max, ratio_s_min, ratio_s_max, flags) as harness._ratio_fields."""
    flags = ""
    k = min(int(n_r), int(result.n_factored))
    if k < n_r:
        flags = "short_factorization"
    if k == 0:
        return 1.0, 1.0, 1.0, 1.0, flags
    packed = result.packed if isinstance(result.packed, np.ndarray) else result.packed.cpu().numpy()
    sigma = np.asarray(sigmas, dtype=np.float64)[:k]
    d = np.sort(np.abs(np.diagonal(packed)[:n_r]))[::-1][:k]
    rd = d / sigma
    r11 = np.triu(packed[:k, :k])
    rs = np.linalg.svd(r11, compute_uv=False) / sigma
    return float(rd.min()), float(rd.max()), float(rs.min()), float(rs.max()), flags
