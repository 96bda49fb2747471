"""CPU oracle for the QRDM / QRDM2 hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it;
the product path (``paper_2106_03138_b200``) never does, and it has no CPU
fallback into this file.

It restates, in plain numpy, the reference's algorithm for the path named in
BASELINE.json ``north_star`` (reference package ``dmqr`` 0.1.0 under
``/root/reference/pkg/src/dmqr``).  Every function cites the reference line
range it follows.  The arithmetic is deliberately the same sequence of numpy
operations as the reference (same reductions, same division/multiplication
order), so the oracle reproduces the reference bit for bit in the same numpy
build; ``tests/test_oracle_golden.py`` pins that against golden vectors made by
running the reference itself (``tests/golden/make_golden.py``).

Beyond the reference it records a per-decision *margin trace* (SURVEY §8d):
how far every comparison that steers the factorization was from flipping.
Parity tests use it to decide where the GPU must agree exactly.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

EPS = float(np.finfo(np.float64).eps)  # rrqr.py:55
TINY = float(np.finfo(np.float64).tiny)

# stop-rule names (rrqr.py:58-63)
STOP_EPS_N, STOP_EPS_SQRT_N, STOP_NONE = "n", "sqrt-n", "none"


# ----------------------------------------------------------------------------
# dense kernels (matrix.py)
# ----------------------------------------------------------------------------

def as_work(a) -> np.ndarray:
    """Validated Fortran-order float64 copy -- matrix.py:24-34 (``dense``)."""
    w = np.array(a, dtype=np.float64, order="F")
    if w.ndim != 2:
        raise ValueError(f"expected a 2-d array, got ndim={w.ndim}")
    if w.size and not np.isfinite(w).all():
        raise ValueError("matrix contains NaN or Inf entries")
    return w


def col_norms(a: np.ndarray) -> np.ndarray:
    """Max-abs-scaled Euclidean column norms -- matrix.py:61-78."""
    if a.ndim == 1:
        a = a[:, None]
    out = np.zeros(a.shape[1])
    if a.shape[0] == 0 or a.shape[1] == 0:
        return out
    scale = np.abs(a).max(axis=0)
    live = scale > 0.0
    if live.any():
        s = a[:, live] / scale[live]
        out[live] = scale[live] * np.sqrt(np.einsum("ij,ij->j", s, s))
    return out


# ----------------------------------------------------------------------------
# reflectors (householder.py)
# ----------------------------------------------------------------------------

def householder(x: np.ndarray):
    """(v, coeff, beta) with (I - coeff v v^T) x = beta e1 -- householder.py:57-79.

    v[0] = 1; beta = -sign(x0)*||x|| (x0 == 0 -> -||x||); x == 0 -> identity.
    No "already triangular" shortcut: x = (x0, 0, ...) still reflects (coeff 2).
    """
    x = np.asarray(x, dtype=np.float64)
    v = np.zeros(x.size)
    v[0] = 1.0
    amax = np.abs(x).max()
    if amax == 0.0:
        return v, 0.0, 0.0
    xs = x / amax
    nrm = amax * math.sqrt(float(xs @ xs))
    beta = -math.copysign(nrm, x[0]) if x[0] != 0.0 else -nrm
    if x.size > 1:
        v[1:] = x[1:] / (x[0] - beta)
    return v, (beta - x[0]) / beta, beta


def reflect_left(v: np.ndarray, coeff: float, c: np.ndarray) -> None:
    """c <- (I - coeff v v^T) c as one rank-1 update -- householder.py:82-89."""
    if coeff == 0.0:
        return
    w = coeff * (v @ c)
    c -= np.outer(v, w)


def wy_factor(vs: list, coeffs: list):
    """Compact (Y, W) with H_1..H_k = I - Y W Y^T -- householder.py:92-114 (larft fwd/col)."""
    mm = vs[0].size
    k = len(vs)
    Y = np.zeros((mm, k), order="F")
    W = np.zeros((k, k), order="F")
    for j in range(k):
        Y[j:, j] = vs[j]
        if j:
            z = Y[j:, :j].T @ vs[j]
            W[:j, j] = -coeffs[j] * (W[:j, :j] @ z)
        W[j, j] = coeffs[j]
    return Y, W


def block_reflect_left(Y: np.ndarray, W: np.ndarray, c: np.ndarray) -> None:
    """c <- (I - Y W^T Y^T) c -- householder.py:117-128 with gemm matrix.py:37-58."""
    t = Y.T @ c
    t = W.T @ t
    prod = Y @ t
    c *= 1.0
    c += -1.0 * prod


# ----------------------------------------------------------------------------
# selector (dm.py)
# ----------------------------------------------------------------------------

def candidates(u: np.ndarray, tau: float, k_dm: int):
    """Seed = first argmax; candidates u_i >= tau*u_seed (i != seed), stable
    descending, first k_dm -- dm.py:81-97."""
    seed = int(np.argmax(u))
    idx = np.flatnonzero(u >= tau * u[seed])
    idx = idx[idx != seed]
    order = np.argsort(-u[idx], kind="stable")
    cand = [int(i) for i in idx[order][:k_dm]]
    return seed, cand


def cosines(c: np.ndarray) -> np.ndarray:
    """Gram-first cosine matrix, upper triangle mirrored, unit diagonal -- dm.py:100-115."""
    nrm = col_norms(c)
    if np.any(nrm == 0.0):
        raise ValueError("cosine matrix undefined: zero column present")
    g = c.T @ c
    inv = 1.0 / nrm
    up = np.triu(g * inv[:, None] * inv[None, :], 1)
    th = up + up.T
    np.fill_diagonal(th, 1.0)
    return th


@dataclass
class Selection:
    cols: list          # selected trailing-relative indices, seed first
    k_max: int
    gamma: float


def select_block(trailing, u, tau, delta, k_dm, use_delta_max, trace=None) -> Selection:
    """Deviation-maximization selection -- dm.py:118-177 (floor test handled by caller)."""
    seed, cand = candidates(u, tau, k_dm)
    k_max = len(cand)
    if trace is not None:
        _trace_candidates(trace, u, tau, k_dm, seed)
    if not cand:
        return Selection([seed], 0, 1.0)
    cols = [seed] + cand
    th = cosines(trailing[:, cols])
    if use_delta_max:
        dlt = tau ** 2 / max(k_max - 1, 1)
        guard = tau ** 2
    else:
        dlt = delta
        guard = None
    chosen = [0]
    rsum = {0: 0.0}
    fmargin = math.inf
    for t in range(1, len(cols)):
        g = np.abs(th[t, chosen])
        fmargin = min(fmargin, float(np.min(np.abs(g - dlt))))
        if not np.all(g < dlt):
            continue
        if guard is not None:
            tot = float(g.sum())
            if tot >= guard or any(rsum[j] + abs(th[j, t]) >= guard for j in chosen):
                continue
            for j in chosen:
                rsum[j] += abs(th[j, t])
            rsum[t] = tot
        chosen.append(t)
    sub = np.abs(th[np.ix_(chosen, chosen)])
    gamma = float(np.min(1.0 - (sub.sum(axis=1) - 1.0)))
    if trace is not None:
        trace["filter"] = min(trace.get("filter", math.inf), fmargin)
    return Selection([cols[t] for t in chosen], k_max, gamma)


def _trace_candidates(trace, u, tau, k_dm, seed):
    """Relative margins of argmax / threshold / ordering / k_dm cut."""
    umax = float(u[seed])
    rest = np.delete(u, seed)
    if rest.size:
        trace["argmax"] = min(trace.get("argmax", math.inf), float((umax - rest.max()) / umax))
        trace["threshold"] = min(trace.get("threshold", math.inf),
                                 float(np.min(np.abs(rest - tau * umax)) / umax))
        s = np.sort(rest[rest >= tau * umax])[::-1]
        if s.size > 1:
            # candidate order only matters up to the k_dm+1-th element
            gaps = np.diff(s[: k_dm + 1])
            gaps = np.abs(gaps[gaps != 0.0]) if np.any(gaps != 0.0) else np.array([])
            if gaps.size:
                trace["order"] = min(trace.get("order", math.inf), float(gaps.min() / umax))
            if np.any(np.diff(s[: k_dm + 1]) == 0.0):
                trace["exact_ties"] = trace.get("exact_ties", 0) + 1


# ----------------------------------------------------------------------------
# decision margins -- not part of the reference
# ----------------------------------------------------------------------------

AMBIGUOUS = 1e3 * EPS  # a decision whose amplified margin is below this may flip


class _Margins:
    """Relative gap of every steering comparison, and the same gap scaled by
    ref_mag/a_max0: trailing quantities carry absolute error ~eps*a_max0, so a
    relative gap g on a quantity of size ref_mag is safe iff g*ref_mag/a_max0
    clears AMBIGUOUS.  ``first_ambiguous`` is the n_s of the first step with a
    decision below that bar (None: the whole run is decided robustly)."""

    def __init__(self, a0: float):
        self.a0 = a0
        self.raw: dict = {}
        self.amp: dict = {}
        self.counts: dict = {}
        self.step_min = math.inf
        self.first_ambiguous = None
        self.per_step: list = []

    def note(self, key: str, gap: float, ref_mag: float):
        g_amp = gap * ref_mag / self.a0 if self.a0 > 0 else gap
        self.raw[key] = min(self.raw.get(key, math.inf), gap)
        self.amp[key] = min(self.amp.get(key, math.inf), g_amp)
        self.step_min = min(self.step_min, g_amp)

    def count(self, key: str, k: int = 1):
        self.counts[key] = self.counts.get(key, 0) + k

    def end_step(self, n_s: int):
        self.per_step.append((n_s, self.step_min))
        if self.first_ambiguous is None and self.step_min <= AMBIGUOUS:
            self.first_ambiguous = n_s
        self.step_min = math.inf

    def summary(self) -> dict:
        out = dict(self.raw)
        out.update({k + "_amp": v for k, v in self.amp.items()})
        out.update(self.counts)
        out["first_ambiguous"] = self.first_ambiguous
        out["per_step"] = self.per_step
        return out


# ----------------------------------------------------------------------------
# the engine (rrqr.py)
# ----------------------------------------------------------------------------

@dataclass
class Step:
    n_s: int
    k_selected: int
    k_accepted: int
    broke_early: bool = False
    fell_back_to_scalar: bool = False
    eps_s: float = 0.0
    gamma: float = 1.0
    k_max: int = 0


@dataclass
class OracleResult:
    packed: np.ndarray
    coeffs: np.ndarray
    forward: np.ndarray
    swaps: list
    rank: int
    steps: list
    n_factored: int
    stopped_early: bool
    counters: tuple            # (rank1, blocked, total) -- rrqr.py:96-110
    norm_trace: list = field(default_factory=list)
    margins: dict = field(default_factory=dict)

    def r_diagonal(self):
        return self.packed.diagonal()[: self.n_factored].copy()


def _eps1(rule: str, epsilon: float, n: int):
    """rrqr.py:75-80."""
    if rule == STOP_EPS_N:
        return epsilon * n
    if rule == STOP_EPS_SQRT_N:
        return epsilon * math.sqrt(n)
    return None


def _downdate(u, uref, work, n_s, n_s1, thr=1e-2):
    """Partial-norm downdate with cancellation guard -- rrqr.py:161-186."""
    n = work.shape[1]
    if not 0 <= n_s < n_s1 <= n:
        raise ValueError(f"bad downdate range [{n_s}, {n_s1}) for n={n}")
    u[:n_s1] = 0.0
    uref[:n_s1] = 0.0
    if n_s1 == n:
        return 0
    r = work[n_s:n_s1, n_s1:]
    sq = u[n_s1:] ** 2 - np.einsum("ij,ij->j", r, r)
    new = np.sqrt(np.maximum(sq, 0.0))
    hit = sq <= thr * uref[n_s1:] ** 2
    nhit = int(np.count_nonzero(hit))
    if nhit:
        loc = np.flatnonzero(hit)
        fresh = col_norms(work[n_s1:, loc + n_s1])
        new[loc] = fresh
        uref[loc + n_s1] = fresh
    u[n_s1:] = new
    return nhit


def _swap(work, u, uref, fwd, swaps, i, j):
    """swap_columns + PartialNorms.swap + Permutation.swap -- matrix.py:81-87,125-132; rrqr.py:131-133."""
    if i == j:
        return
    tmp = work[:, i].copy()
    work[:, i] = work[:, j]
    work[:, j] = tmp
    u[i], u[j] = u[j], u[i]
    uref[i], uref[j] = uref[j], uref[i]
    fwd[i], fwd[j] = fwd[j], fwd[i]
    swaps.append((i, j))


def swap_plan(base: int, targets: list) -> list:
    """The exact transposition sequence of _move_selected_to_front -- rrqr.py:294-312."""
    pos = list(targets)
    out = []
    for i in range(len(pos)):
        tgt = base + i
        src = pos[i]
        if src == tgt:
            continue
        out.append((tgt, src))
        for h in range(i + 1, len(pos)):
            if pos[h] == tgt:
                pos[h] = src
                break
    return out


def qrdm_engine(A, tau=0.15, delta=0.9, k_dm=64, use_delta_max=False,
                stop_rule=STOP_EPS_N, epsilon=EPS, break_check=True,
                trace_norms=False, margins=False, max_steps=0) -> OracleResult:
    """QRDM (break_check=False) / QRDM2 (True) -- rrqr.py:315-423 (+ 426-456)."""
    if not 0.0 < tau <= 1.0:
        raise ValueError(f"tau must be in (0, 1], got {tau}")
    if not 0.0 <= delta < 1.0:
        raise ValueError(f"delta must be in [0, 1), got {delta}")
    if k_dm < 1:
        raise ValueError(f"k_dm must be >= 1, got {k_dm}")
    work = as_work(A)
    m, n = work.shape
    fwd = np.arange(n, dtype=np.intp)
    swaps: list = []
    u = col_norms(work)
    uref = u.copy()
    a0 = float(u.max(initial=0.0))
    floor = n * EPS * a0
    kmax = min(m, n)
    coeffs = np.zeros(kmax)
    rank1 = blocked = 0.0
    total = 2.0 * m * n
    steps: list = []
    ntrace: list = []
    mg = _Margins(a0) if margins else None
    eps1 = _eps1(stop_rule, epsilon, n)
    rank = None
    n_s = 0
    while n_s < kmax:
        if max_steps and len(steps) >= max_steps:  # debug: partial factorization
            break
        ut = u[n_s:]
        umax = float(ut.max())
        # stop test -- rrqr.py:189-203, 336-338
        if eps1 is not None:
            lhs = math.sqrt(n - n_s) * umax
            rhs = eps1 * a0
            if mg is not None and rhs > 0:
                mg.note("stop", abs(lhs - rhs) / rhs, umax)
            if lhs <= rhs:
                rank = n_s
                if mg is not None:
                    mg.end_step(n_s)
                break
        if mg is not None and floor > 0:
            mg.note("floor", abs(umax - floor) / floor, umax)
        if ut.size == 0 or umax <= floor:
            # scalar fallback -- rrqr.py:219-235, 343-353
            s = n_s
            j = s + int(np.argmax(u[s:]))
            if mg is not None:
                mg.count("fallback_steps")
                rest = np.delete(u[s:], j - s)
                if rest.size:
                    mg.note("argmax", float((umax - rest.max()) / umax) if umax > 0 else 0.0, umax)
            _swap(work, u, uref, fwd, swaps, s, j)
            v, cf, beta = householder(work[s:, s])
            coeffs[s] = cf
            if s + 1 < n:
                reflect_left(v, cf, work[s:, s + 1:])
                rank1 += 4.0 * (m - s) * (n - s - 1)
                total += 4.0 * (m - s) * (n - s - 1)
            work[s, s] = beta
            work[s + 1:, s] = v[1:]
            total += 4.0 * (m - s) + (n - s)
            nh = _downdate(u, uref, work, s, s + 1)
            total += 4.0 * (n - s - 1)
            if trace_norms:
                _norm_check(ntrace, u, work, s + 1, a0)
            steps.append(Step(s, 1, 1, fell_back_to_scalar=True))
            if mg is not None:
                mg.count("guard_recomputes", nh)
                mg.end_step(s)
            n_s += 1
            continue

        tr: dict | None = {} if mg is not None else None
        sel = select_block(work[n_s:, n_s:], ut, tau, delta, k_dm, use_delta_max, tr)
        if tr:
            for key, val in tr.items():
                if key == "exact_ties":
                    mg.count("exact_ties", val)
                    mg.note("exact_ties", 0.0, umax)
                elif key == "filter":  # cosines carry error ~eps*a0/||c_j||, ||c_j|| >= tau*umax
                    mg.note(key, val, tau * umax)
                else:
                    mg.note(key, val, umax)
        k_s = min(len(sel.cols), kmax - n_s)
        total += (m - n_s) * (sel.k_max + 1) ** 2
        eps_s = tau * float(u[n_s:].max())
        for (a, b) in swap_plan(n_s, [n_s + r for r in sel.cols[:k_s]]):
            _swap(work, u, uref, fwd, swaps, a, b)

        vs, cfs = [], []
        broke = False
        for l in range(k_s):
            col = n_s + l
            v, cf, beta = householder(work[col:, col])
            coeffs[col] = cf
            if col + 1 < n_s + k_s:
                reflect_left(v, cf, work[col:, col + 1:n_s + k_s])
                fl = 4.0 * (m - col) * (n_s + k_s - col - 1)
                rank1 += fl
                total += fl
            work[col, col] = beta
            work[col + 1:, col] = v[1:]
            total += 4.0 * (m - col)
            vs.append(v)
            cfs.append(cf)
            if break_check and l + 1 < k_s:
                nxt = col + 1
                r = float(col_norms(work[nxt:, nxt])[0])
                if mg is not None and eps_s > 0:
                    mg.note("break", abs(r - eps_s) / eps_s, eps_s)
                if r < eps_s:
                    broke = True
                    break
        l_acc = len(vs)
        if n_s + k_s < n:
            Y, W = wy_factor(vs, cfs)
            total += 2.0 * (m - n_s) * l_acc ** 2
            block_reflect_left(Y, W, work[n_s:, n_s + k_s:])
            fl = (4.0 * (m - n_s) * l_acc + 2.0 * l_acc ** 2) * (n - n_s - k_s)
            blocked += fl
            total += fl
        n_s1 = n_s + l_acc
        nh = _downdate(u, uref, work, n_s, n_s1)
        total += 2.0 * l_acc * (n - n_s1) if n_s1 < n else 0.0
        if trace_norms:
            _norm_check(ntrace, u, work, n_s1, a0)
        steps.append(Step(n_s, k_s, l_acc, broke, False, eps_s, sel.gamma, sel.k_max))
        if mg is not None:
            mg.count("guard_recomputes", nh)
            mg.end_step(n_s)
        n_s = n_s1

    stopped = rank is not None
    n_fact = n_s if stopped else min(n_s, kmax)
    if rank is None:
        if stop_rule == STOP_NONE:
            d = work.diagonal()[:n_fact]
            rank = int(np.count_nonzero(np.abs(d) > EPS * n * a0))  # rrqr.py:206-208
        else:
            rank = n_fact
    return OracleResult(work, coeffs, fwd, swaps, rank, steps, n_fact, stopped,
                        (rank1, blocked, total), ntrace, mg.summary() if mg is not None else {})


def _norm_check(trace, u, work, n_s1, scale):
    """rrqr.py:211-216."""
    if n_s1 >= work.shape[1]:
        return
    direct = col_norms(work[n_s1:, n_s1:])
    den = np.maximum(np.maximum(direct, EPS * scale), TINY)
    trace.append(float(np.max(np.abs(u[n_s1:] - direct) / den)))


def qrdm(A, **kw) -> OracleResult:
    """rrqr.py:426-440."""
    return qrdm_engine(A, break_check=False, **kw)


def qrdm2(A, **kw) -> OracleResult:
    """rrqr.py:443-456."""
    return qrdm_engine(A, break_check=True, **kw)


def qrp(A, stop_rule=STOP_EPS_N, epsilon=EPS, trace_norms=False, margins=False, max_steps=0) -> OracleResult:
    """QR with greedy column pivoting -- rrqr.py:238-291 (one _scalar_step,
    rrqr.py:219-235, then downdate_norms(s, s+1) per column)."""
    work = as_work(A)
    m, n = work.shape
    fwd = np.arange(n, dtype=np.intp)
    swaps: list = []
    u = col_norms(work)
    uref = u.copy()
    a0 = float(u.max(initial=0.0))
    kmax = min(m, n)
    coeffs = np.zeros(kmax)
    rank1 = 0.0
    total = 2.0 * m * n
    steps: list = []
    ntrace: list = []
    mg = _Margins(a0) if margins else None
    eps1 = _eps1(stop_rule, epsilon, n)
    rank = None
    done = 0
    for s in range(kmax):
        if max_steps and s >= max_steps:
            break
        umax = float(u[s:].max())
        if eps1 is not None:  # check_stop, rrqr.py:189-203
            lhs = math.sqrt(n - s) * umax
            rhs = eps1 * a0
            if mg is not None and rhs > 0:
                mg.note("stop", abs(lhs - rhs) / rhs, umax)
            if lhs <= rhs:
                rank = s
                if mg is not None:
                    mg.end_step(s)
                break
        j = s + int(np.argmax(u[s:]))
        if mg is not None:
            rest = np.delete(u[s:], j - s)
            if rest.size:
                mg.note("argmax", float((umax - rest.max()) / umax) if umax > 0 else 0.0, umax)
        _swap(work, u, uref, fwd, swaps, s, j)
        v, cf, beta = householder(work[s:, s])
        coeffs[s] = cf
        if s + 1 < n:
            reflect_left(v, cf, work[s:, s + 1:])
            rank1 += 4.0 * (m - s) * (n - s - 1)
            total += 4.0 * (m - s) * (n - s - 1)
        work[s, s] = beta
        work[s + 1:, s] = v[1:]
        total += 4.0 * (m - s) + (n - s)
        nh = _downdate(u, uref, work, s, s + 1)
        total += 4.0 * (n - s - 1)
        if trace_norms:
            _norm_check(ntrace, u, work, s + 1, a0)
        steps.append(Step(s, 1, 1))
        if mg is not None:
            mg.count("guard_recomputes", nh)
            mg.end_step(s)
        done = s + 1
    stopped = rank is not None
    if rank is None:
        if stop_rule == STOP_NONE:
            rank = int(np.count_nonzero(np.abs(work.diagonal()[:done]) > EPS * n * a0))  # rrqr.py:206-208
        else:
            rank = done
    return OracleResult(work, coeffs, fwd, swaps, rank, steps, done, stopped, (rank1, 0.0, total), ntrace,
                        mg.summary() if mg is not None else {})


def explicit_q(packed: np.ndarray, coeffs: np.ndarray, n_factored: int, ncols=None):
    """Q (m x ncols, default m) by backward reflector accumulation -- rrqr.py:459-480."""
    m = packed.shape[0]
    ncols = m if ncols is None else ncols
    Q = np.eye(m, ncols, order="F")
    for s in range(n_factored - 1, -1, -1):
        v = np.empty(m - s)
        v[0] = 1.0
        v[1:] = packed[s + 1:, s]
        t = coeffs[s]
        if t != 0.0:
            w = t * (v @ Q[s:, :])
            Q[s:, :] -= np.outer(v, w)
    return Q


def r_factor(packed: np.ndarray, n_factored: int) -> np.ndarray:
    """R = packed with the factored sub-diagonals zeroed (raw trailing block kept) -- rrqr.py:477-480."""
    R = np.asfortranarray(packed.copy())
    for j in range(min(n_factored, packed.shape[1])):
        R[j + 1:, j] = 0.0
    return R
