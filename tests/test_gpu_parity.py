"""GPU parity: the CUDA path (through the C-ABI) vs the reference's golden
vectors and the live CPU oracle.  Needs a B200 (``-m gpu``)."""

import functools

import numpy as np
import pytest
from threadpoolctl import threadpool_limits

import golden_cases as G
import parity
from oracle import qrdm_oracle as O

pytestmark = pytest.mark.gpu

GOLDEN = [c for c in G.case_names() if not c.startswith(("cfg2s", "cfg4s"))]


def _gpu(name_or_A, algo="qrdm2", **kw):
    from paper_2106_03138_b200 import DMParams, StopCriterion, StopRule, qrdm, qrdm2, qrp

    stop = StopCriterion(StopRule(kw.get("stop_rule", "n")))
    if algo == "qrp":
        return qrp(name_or_A, stop=stop, trace_norms=kw.get("trace_norms", False))
    params = DMParams(**{k: kw[k] for k in ("tau", "delta", "k_dm", "use_delta_max") if k in kw})
    fn = qrdm2 if algo == "qrdm2" else qrdm
    return fn(name_or_A, params=params, stop=stop, trace_norms=kw.get("trace_norms", False))


def _steps(log):
    return [(s.n_s, s.k_selected, s.k_accepted, s.broke_early, s.fell_back_to_scalar,
             s.k_max if not s.fell_back_to_scalar else -1) for s in log]


def _compare(A, res, ref, label, require_full=False, min_cut=0):
    """Exact decisions up to the first ambiguous one (all of them when the run is
    robust, or when ``require_full``: inputs the reference itself decides stably,
    SURVEY App. B), at least ``min_cut`` columns, |diag R| to 1e-10 there,
    residual/orthogonality <= 50 n eps always."""
    m, n = A.shape
    cut, full = parity.robust_prefix(ref)
    assert cut >= min(min_cut, ref.n_factored), f"{label}: robust prefix {cut} < {min_cut} (vacuous gate)"
    if require_full:
        cut, full = ref.n_factored, True
    assert np.array_equal(res.perm.forward[:cut], ref.forward[:cut]), f"{label}: pivots differ before column {cut}"
    want = [s for s in ref.steps if s.n_s < cut]
    assert _steps(res.step_log[:len(want)]) == _steps(want), f"{label}: step log differs before column {cut}"
    ok, worst = parity.diag_close(res.r_diagonal()[:cut], ref.r_diagonal()[:cut], max(m, n))
    assert ok, f"{label}: |diag R| off by {worst:.3g} x tolerance"
    for a, b in zip(res.step_log[:len(want)], want):
        # eps_s = tau * (downdated max norm): downdating amplifies rounding
        assert a.eps_s == pytest.approx(b.eps_s, rel=1e-9, abs=0)
        # gamma (diagnostic) sums |cosines| of possibly ill-conditioned trailing columns
        assert a.gamma == pytest.approx(b.gamma, rel=1e-6, abs=1e-9)
    if full:
        assert np.array_equal(res.perm.forward, ref.forward), f"{label}: permutation differs"
        assert res.perm.swaps == [tuple(map(int, s)) for s in ref.swaps], f"{label}: swap log differs"
        assert res.rank == ref.rank, (label, res.rank, ref.rank)
        assert res.n_factored == ref.n_factored and res.stopped_early == ref.stopped_early
        assert _steps(res.step_log) == _steps(ref.steps), f"{label}: step log differs"
        rc = res.counters
        assert (rc.rank1_flops, rc.blocked_flops, rc.total_flops) == pytest.approx(ref.counters, rel=0, abs=0)
    if m and n:
        resid, orth = parity.residuals(A, res)
        bound = 50 * max(m, n) * O.EPS
        assert resid <= bound, f"{label}: residual {resid:.3g} > {bound:.3g}"
        assert orth <= bound, f"{label}: orthogonality {orth:.3g} > {bound:.3g}"
    return cut, full


@pytest.fixture(params=["fused", "steps"])
def small_path(request, monkeypatch):
    """Small inputs (m <= 256, n <= 512) run the fused per-matrix kernel by
    default (small.cuh); "steps" forces the per-step kernels (DMQR_NO_FUSED)."""
    if request.param == "steps":
        monkeypatch.setenv("DMQR_NO_FUSED", "1")
    return request.param


@functools.lru_cache(maxsize=None)
def _golden_oracle(name):
    """The oracle's run (with margins) of a golden case, shared by both small paths."""
    meta = G.index()["cases"][name]
    A = G.case_input(name)
    kw = G.oracle_kwargs(name)
    with threadpool_limits(1):
        if meta["algo"] == "qrp":
            return O.qrp(A, margins=True, stop_rule=kw["stop_rule"])
        return (O.qrdm2 if meta["algo"] == "qrdm2" else O.qrdm)(A, margins=True, **kw)


@pytest.mark.parametrize("name", GOLDEN)
def test_golden_case(name, small_path):
    meta = G.index()["cases"][name]
    A = G.case_input(name)
    kw = G.oracle_kwargs(name)
    res = _gpu(A, meta["algo"], **kw)
    ref = _golden_oracle(name)
    # the oracle itself is pinned to the golden vectors (test_oracle_golden.py)
    assert np.array_equal(ref.forward, G.case_field(name, "forward"))
    # BASELINE cfg1 is stable under 1-ulp input perturbation:
    # with an active stop rule the whole run must match, rank included (with
    # StopRule.NONE the run continues into the 1e-18 noise block, whose pivots
    # are round-off-determined).  Exact ties (identity, duplicate
    # columns, Kahan) have a zero margin by construction; everything else must be
    # robust for at least its first pivot.
    tie = name.split("/")[-1].startswith(("identity", "duplicate", "kahan")) or "/kahan" in name
    _compare(A, res, ref, name, require_full=name in ("cfg1/qrdm", "cfg1/qrdm2"), min_cut=0 if tie else 1)


@pytest.mark.parametrize("seed", range(12))
def test_random_vs_oracle(seed, small_path):
    rng = np.random.default_rng(1000 + seed)
    m = int(rng.integers(40, 400))
    n = int(rng.integers(40, 400))
    kind = seed % 3
    if kind == 0:
        A = rng.standard_normal((m, n))
    elif kind == 1:
        r = int(rng.integers(1, min(m, n)))
        A = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    else:
        A = rng.standard_normal((m, n)) * np.logspace(0, -10, n)[rng.permutation(n)]
    algo = "qrdm2" if seed % 2 == 0 else "qrdm"
    res = _gpu(A, algo)
    with threadpool_limits(1):
        ref = (O.qrdm2 if algo == "qrdm2" else O.qrdm)(A, margins=True)
    _compare(A, res, ref, f"random{seed}")


@pytest.mark.parametrize("seed", range(8))
def test_qrp_random_vs_oracle(seed):
    """qrp on the blocked scalar-pivot engine: shapes across block boundaries
    (64 columns per block), tall / wide / rank-deficient / graded inputs."""
    rng = np.random.default_rng(2380 + seed)
    m = int(rng.integers(30, 700))
    n = int(rng.integers(30, 700))
    kind = seed % 4
    if kind == 0:
        A = rng.standard_normal((m, n))
    elif kind == 1:
        r = int(rng.integers(1, min(m, n)))
        A = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    elif kind == 2:
        A = rng.standard_normal((m, n)) * np.logspace(0, -12, n)[rng.permutation(n)]
    else:
        A = rng.standard_normal((m, n)) * 10.0 ** rng.uniform(-6, 0, n)
    stop_rule = ("n", "none", "sqrt-n", "n")[seed % 4]
    res = _gpu(A, "qrp", stop_rule=stop_rule)
    with threadpool_limits(1):
        ref = O.qrp(A, margins=True, stop_rule=stop_rule)
    _compare(A, res, ref, f"qrp-random{seed}")


def test_qrp_guard_overflow_block_end():
    """Many near-parallel columns: the first reflector sends most norms under the
    guard at once (> 64 guards), so the block ends and they are recomputed from
    the updated matrix (rrqr.py:178-184 semantics)."""
    rng = np.random.default_rng(77)
    x = rng.standard_normal(300)
    A = np.outer(x, 1.0 + 0.1 * rng.standard_normal(200)) + 1e-7 * rng.standard_normal((300, 200))
    for algo in ("qrp", "qrdm2"):
        res = _gpu(A, algo, stop_rule="none")
        with threadpool_limits(1):
            ref = (O.qrp(A, margins=True, stop_rule="none") if algo == "qrp"
                   else O.qrdm2(A, margins=True, stop_rule="none"))
        _compare(A, res, ref, f"guard-overflow-{algo}")


def test_qrp_midsize_blocks():
    """1200 x 900: 15 blocks of the delayed-update engine against the oracle."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((1200, 900)) * np.logspace(0, -9, 900)
    res = _gpu(A, "qrp")
    with threadpool_limits(1):
        ref = O.qrp(A, margins=True)
    _compare(A, res, ref, "qrp-midsize")


def test_qrp_trace_norms():
    rng = np.random.default_rng(40)
    A = rng.standard_normal((120, 90))
    res = _gpu(A, "qrp", stop_rule="none", trace_norms=True)
    with threadpool_limits(1):
        ref = O.qrp(A, stop_rule="none", trace_norms=True)
    assert len(res.norm_trace) == len(ref.norm_trace)
    assert max(res.norm_trace) <= 1e-10


def test_registry_run_algorithm_on_device():
    """registry.run_algorithm (harness.py:188-198 surface) dispatches to the device engine."""
    from paper_2106_03138_b200 import DMParams, StopCriterion, qrp, registry

    rng = np.random.default_rng(3)
    A = rng.standard_normal((90, 70))
    a = registry.run_algorithm("qrp", A, DMParams(), StopCriterion())
    b = qrp(A)
    assert np.array_equal(a.packed, b.packed) and np.array_equal(a.perm.forward, b.perm.forward)
    ref_style = registry.register({})
    c = ref_style["qrdm2_b200"](A, params=DMParams(), stop=StopCriterion())
    assert c.rank == registry.run_algorithm("qrdm2", A, DMParams(), StopCriterion()).rank


def test_trace_norms_within_1e10():
    rng = np.random.default_rng(39)
    A = rng.standard_normal((250, 180))
    res = _gpu(A, "qrdm2", k_dm=8, stop_rule="none", trace_norms=True)
    assert res.norm_trace and max(res.norm_trace) <= 1e-10


def test_errors():
    from paper_2106_03138_b200 import DMParams, qrdm2

    with pytest.raises(ValueError):
        qrdm2(np.ones(3))
    bad = np.ones((4, 4))
    bad[1, 2] = np.nan
    with pytest.raises(ValueError):
        qrdm2(bad)
    bad[1, 2] = np.inf
    with pytest.raises(ValueError):
        qrdm2(bad)
    with pytest.raises(ValueError):
        DMParams(tau=0.0)


def test_input_not_mutated_and_torch_input():
    import torch

    from paper_2106_03138_b200 import qrdm2

    rng = np.random.default_rng(5)
    A = rng.standard_normal((70, 50))
    A0 = A.copy()
    r1 = qrdm2(A)
    assert np.array_equal(A, A0)
    r2 = qrdm2(torch.from_numpy(A).cuda())
    assert np.array_equal(r1.perm.forward, r2.perm.forward)
    assert np.array_equal(r1.packed, r2.packed)


def test_empty_and_degenerate_shapes():
    from paper_2106_03138_b200 import qrdm, qrdm2

    for shape in [(0, 0), (0, 5), (5, 0)]:
        r = qrdm2(np.zeros(shape))
        assert r.rank == 0 and r.n_factored == 0 and r.step_log == []
    r = qrdm(np.zeros((4, 3)))
    assert r.rank == 0


def test_deterministic_repeat():
    from paper_2106_03138_b200 import qrdm2

    rng = np.random.default_rng(11)
    A = rng.standard_normal((300, 260))
    a, b = qrdm2(A), qrdm2(A)
    assert np.array_equal(a.packed, b.packed) and np.array_equal(a.coeffs, b.coeffs)


@pytest.mark.parametrize("name", ["cfg2s/1024", "cfg4s/8192x256"])
def test_midsize_golden(name):
    test_golden_case(name, "fused")  # (too large for the fused kernel: per-step kernels)


def test_batched_equals_single_and_oracle():
    """cfg3-style batch through dmqr_qrdm_batched_f64 (concurrent lanes, replayed
    step graphs): each matrix takes the single-matrix factorization's decisions,
    equal factors to rounding, and matches the oracle on the robust prefix."""
    from paper_2106_03138_b200 import inputs, qrdm2
    from paper_2106_03138_b200.batch import factorize_batch

    B = inputs.cfg3(seed=3, batch=6)
    f = factorize_batch(B, lanes=4)
    for i in range(B.shape[0]):
        r = f.result(i)
        s = qrdm2(B[i])
        assert np.array_equal(r.perm.forward, s.perm.forward) and r.rank == s.rank
        assert [(a.n_s, a.k_selected, a.k_accepted) for a in r.step_log] == \
            [(a.n_s, a.k_selected, a.k_accepted) for a in s.step_log]
        # the batch replays a whole-matrix step graph per lane (split-K counts
        # sized for the full matrix), so sums may associate differently
        scale = np.abs(s.packed).max()
        assert np.abs(r.packed - s.packed).max() <= 1e-12 * scale
        assert np.allclose(r.coeffs, s.coeffs, rtol=1e-12, atol=1e-14)
        with threadpool_limits(1):
            ref = O.qrdm2(B[i], margins=True)
        _compare(B[i], r, ref, f"cfg3[{i}]")


def test_streamed_packed_equals_device_copy():
    """dmqr_qrdm_stream_f64 (the qrdm2 default) hands back the same packed factor
    as a device-side result copied afterwards."""
    from paper_2106_03138_b200 import qrdm2

    rng = np.random.default_rng(21)
    A = rng.standard_normal((1200, 1000))
    a = qrdm2(A)
    b = qrdm2(A, device=True)
    assert np.array_equal(a.packed, b.packed.cpu().numpy())
    assert np.array_equal(a.perm.forward, b.perm.forward)


@pytest.mark.parametrize("shape", [(1100, 1000), (6000, 700)])
def test_lookahead_matches_serial_schedule(shape, monkeypatch):
    """The look-ahead schedule (panel || rest of the previous update, Wt from
    G = Q1^T C) against the serial one on the same input: identical decisions,
    factors equal to rounding.  (6000 rows starts on the Householder panel and
    switches schedule once m' <= 4096.)"""
    from paper_2106_03138_b200 import qrdm2

    rng = np.random.default_rng(22)
    m, n = shape
    A = rng.standard_normal((m, n)) * np.logspace(0, -3, n)[rng.permutation(n)]
    la = qrdm2(A)
    monkeypatch.setenv("DMQR_NO_LOOKAHEAD", "1")
    se = qrdm2(A)
    assert np.array_equal(la.perm.forward, se.perm.forward) and la.rank == se.rank
    assert [(s.n_s, s.k_selected, s.k_accepted) for s in la.step_log] == \
        [(s.n_s, s.k_selected, s.k_accepted) for s in se.step_log]
    scale = np.abs(se.packed).max()
    assert np.abs(la.packed - se.packed).max() <= 1e-10 * scale
    resid, orth = parity.residuals(A, la)
    assert resid <= 50 * max(m, n) * O.EPS and orth <= 50 * max(m, n) * O.EPS


# ----------------------------------------------------------------------------
# BASELINE full sizes: size-independent properties, computed on the device
# (Q from the blocked dmqr_form_q_f64; products by torch / cuBLAS in fp64 --
# test harness only)
# ----------------------------------------------------------------------------

def _device_residuals(A_dev, res):
    """||A P - Q R||_F / ||A||_F and ||Q^T Q - I||_F with thin Q (m x min(m, n))."""
    import torch
    from paper_2106_03138_b200 import form_q

    m, n = A_dev.shape
    packed = res.packed  # device (m x n) view
    k = min(m, n)
    Q = form_q(packed, res.coeffs, res.n_factored, qcols=k)
    R = torch.triu(packed[:k, :].clone())
    nf = res.n_factored
    if nf < k:  # the raw trailing block below row nf (columns >= nf) is part of R
        R[nf:, nf:] = packed[nf:k, nf:]
    perm = torch.as_tensor(np.asarray(res.perm.forward), device=A_dev.device)
    AP = A_dev[:, perm]
    if m > k:  # rows past k of the trailing block: Q is thin, so fold them in explicitly
        # A P = Q_full R_full; with the thin Q the rows >= k of R (only in columns >= nf) are lost:
        # require them to be zero-sized (nf == k) for tall inputs
        assert nf == k or m == k
    resid = (torch.linalg.matrix_norm(AP - Q @ R) / torch.linalg.matrix_norm(A_dev)).item()
    orth = torch.linalg.matrix_norm(Q.T @ Q - torch.eye(k, dtype=Q.dtype, device=Q.device)).item()
    return resid, orth


@pytest.mark.parametrize("algo", ["qrdm2", "qrdm"])
def test_cfg2_full_size_vs_oracle(algo):
    """BASELINE cfg2 (4096^2 N(0,1), seed 1) at full size: the same permutation
    and rank as the CPU oracle (all host BLAS threads), residual and
    orthogonality <= 50 n eps."""
    import torch
    from paper_2106_03138_b200 import inputs, qrdm, qrdm2

    A = inputs.cfg2(seed=1)
    res = (qrdm2 if algo == "qrdm2" else qrdm)(A, device=True)
    ref = (O.qrdm2 if algo == "qrdm2" else O.qrdm)(A, margins=True)
    # cfg2 is decided stably by the reference (identical under a
    # 1-ulp perturbation): the whole run must match
    assert np.array_equal(np.asarray(res.perm.forward), ref.forward) and res.rank == ref.rank
    assert _steps(res.step_log) == _steps(ref.steps)
    ok, worst = parity.diag_close(res.r_diagonal(), ref.r_diagonal(), 4096)
    assert ok, f"|diag R| off by {worst:.3g} x tolerance"
    assert res.rank == 4096 and len(res.step_log) == len(ref.steps)
    resid, orth = _device_residuals(torch.as_tensor(A, device="cuda"), res)
    bound = 50 * 4096 * O.EPS
    assert resid <= bound and orth <= bound, (resid, orth)


def test_cfg4_full_size_properties():
    """BASELINE cfg4 (65536 x 1024 tall, graded columns) at full size on the device."""
    import torch
    from paper_2106_03138_b200 import inputs, qrdm2

    A = inputs.device_cfg("cfg4", seed=4)
    res = qrdm2(A, device=True)
    assert res.rank == 1024 and not res.stopped_early
    resid, orth = _device_residuals(A, res)
    bound = 50 * 65536 * O.EPS
    assert resid <= bound and orth <= bound, (resid, orth)


@pytest.mark.parametrize("algo", ["qrdm2", "qrp"])
def test_cfg5_full_size_properties(algo):
    """BASELINE cfg5 (16384^2 graded, near-collinear columns) at full size: the
    rank-revealing stop (sqrt(n - k) max trailing norm <= n eps ||a||_max,
    rrqr.py:189-203), residual and orthogonality <= 50 n eps."""
    import torch
    from paper_2106_03138_b200 import inputs, qrdm2, qrp

    n = 16384
    A = inputs.device_cfg("cfg5", seed=4)
    res = (qrdm2 if algo == "qrdm2" else qrp)(A, device=True)
    assert res.stopped_early and 9000 < res.rank < 10500, res.rank
    k = res.rank
    a0 = torch.linalg.vector_norm(A, dim=0).max().item()
    trail = torch.linalg.vector_norm(res.packed[k:, k:], dim=0).max().item()
    assert np.sqrt(n - k) * trail <= n * O.EPS * a0 * (1 + 1e-6), (trail, a0)
    resid, orth = _device_residuals(A, res)
    bound = 50 * n * O.EPS
    assert resid <= bound and orth <= bound, (resid, orth)


# ----------------------------------------------------------------------------
# rank-revealing quality (acceptance criterion 2, test_acceptance.py:108-132):
# |d_i| / sigma_i within [1e-1, 1e1] over the numerical rank -- on the fixture
# suite (sigma by LAPACK) and, beyond the reference's 512-column SVD cap, on
# device-built matrices of known spectrum
# ----------------------------------------------------------------------------

def test_criterion2_factor10_ratios_fixture_suite():
    import fixture_suite
    from paper_2106_03138_b200 import DMParams, StopCriterion, StopRule, qrdm2
    from paper_2106_03138_b200.diagnostics import ratio_fields

    bad = []
    for name, A in fixture_suite.suite():
        s = np.linalg.svd(A, compute_uv=False)
        nr = int(np.count_nonzero(s > max(A.shape) * O.EPS * (s[0] if s.size else 0.0)))
        if nr == 0:
            continue
        res = qrdm2(A, params=DMParams(), stop=StopCriterion(StopRule.NONE))
        d_lo, d_hi, s_lo, s_hi, flags = ratio_fields(res, s, nr)
        if d_lo < 1e-1 or d_hi > 1e1:
            bad.append((name, d_lo, d_hi))
        assert s_hi <= 1.0 + 1e-8  # interlacing: sigma_i(R11) <= sigma_i(A)
    assert not bad, bad


@pytest.mark.parametrize("n", [2048, 4096])
def test_factor10_ratios_known_spectrum_beyond_cpu_cap(n):
    """cfg1's recipe scaled up on the device: A = U diag(sigma) V^T, Haar U, V,
    sigma_i = 10^(-4 (i-1)/(r-1)) for i <= r = 3n/4, 1e-18 after: qrdm2 must
    reveal rank r (up to round-off-level columns) with |d_i| / sigma_i within
    [1e-1, 1e1] over the first r."""
    import torch
    from paper_2106_03138_b200 import qrdm2

    g = torch.Generator(device="cuda")
    g.manual_seed(n)

    def haar(k):
        q, r = torch.linalg.qr(torch.randn(k, k, generator=g, dtype=torch.float64, device="cuda"))
        return q * torch.sign(torch.diagonal(r))

    r = 3 * n // 4
    sig = torch.full((n,), 1e-18, dtype=torch.float64, device="cuda")
    sig[:r] = 10.0 ** (-4.0 * torch.arange(r, dtype=torch.float64, device="cuda") / (r - 1))
    A = (haar(n) * sig) @ haar(n).T
    res = qrdm2(A, device=True)
    # the 1e-18 tail sits below the product's own round-off (~eps ||A||), so the
    # stop rule may keep a few noise-level columns past r
    assert r <= res.rank <= r + n // 256, (res.rank, r)
    d = torch.sort(torch.abs(torch.diagonal(res.packed)[:r]), descending=True).values
    ratios = (d / sig[:r]).cpu().numpy()
    assert ratios.min() >= 1e-1 and ratios.max() <= 1e1, (ratios.min(), ratios.max())


def test_batched_graph_lanes_with_fallback_runs(small_path):
    """Batched lanes (replayed step graphs) on inputs whose factorization falls
    back to scalar pivoting (the blocked scalar-pivot engine runs between graph
    replays): same decisions as the single-matrix calls, oracle on the robust prefix."""
    from paper_2106_03138_b200 import DMParams, StopCriterion, StopRule, qrdm2
    from paper_2106_03138_b200.batch import factorize_batch

    rng = np.random.default_rng(36)
    B = np.stack([rng.standard_normal((48, 5)) @ rng.standard_normal((5, 40)) * (1 + i) for i in range(8)])
    none = StopCriterion(StopRule.NONE)  # past the rank the norms sit under the floor: scalar-pivot runs
    f = factorize_batch(B, DMParams(), none, True, lanes=3)
    saw_fallback = False
    for i in range(B.shape[0]):
        r = f.result(i)
        s = qrdm2(B[i], stop=none)
        saw_fallback |= any(st.fell_back_to_scalar for st in s.step_log)
        assert np.array_equal(r.perm.forward, s.perm.forward) and r.rank == s.rank
        assert [(a.n_s, a.k_selected, a.k_accepted, a.fell_back_to_scalar) for a in r.step_log] == \
            [(a.n_s, a.k_selected, a.k_accepted, a.fell_back_to_scalar) for a in s.step_log]
        with threadpool_limits(1):
            ref = O.qrdm2(B[i], margins=True, stop_rule="none")
        _compare(B[i], r, ref, f"batch-fallback[{i}]")
    assert saw_fallback


@pytest.mark.parametrize("wait_ns", ["0", None])
def test_tall_panel_helpers_and_their_fallback(wait_ns, monkeypatch):
    """Tall panels (m' > 16 x 256, serial schedule) take their row passes from
    k_panel_helper; with no wait (DMQR_HELPER_WAIT_NS=0) the cluster abandons
    them and streams its own rows -- the path a serialised launch takes.  Both
    must give the no-helper factorization's decisions and factors to rounding."""
    from paper_2106_03138_b200 import qrdm2

    rng = np.random.default_rng(44)
    A = rng.standard_normal((9000, 300)) * np.logspace(0, -4, 300)[rng.permutation(300)]
    monkeypatch.setenv("DMQR_NO_HELPERS", "1")
    base = qrdm2(A)
    monkeypatch.delenv("DMQR_NO_HELPERS")
    if wait_ns is not None:
        monkeypatch.setenv("DMQR_HELPER_WAIT_NS", wait_ns)
    res = qrdm2(A)
    assert np.array_equal(res.perm.forward, base.perm.forward) and res.rank == base.rank
    scale = np.abs(base.packed).max()
    assert np.abs(res.packed - base.packed).max() <= 1e-10 * scale
    resid, orth = parity.residuals(A, res)
    assert resid <= 50 * 9000 * O.EPS and orth <= 50 * 9000 * O.EPS


@pytest.mark.parametrize("n", [1536, 2500])
def test_pmode_lookahead_matches_default(monkeypatch, n):
    """Opt-in P-mode look-ahead (DMQR_PMODE: k_spare forms P^T C from the panel's
    start, k_trail_w folds R1^-T into MT): same decisions as the default schedule,
    factor equal to rounding of a cond(R1)-scaled product."""
    from paper_2106_03138_b200 import qrdm2

    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n)) * np.logspace(0, -6, n)[rng.permutation(n)]
    base = qrdm2(A)
    monkeypatch.setenv("DMQR_PMODE", "1")
    res = qrdm2(A)
    assert np.array_equal(res.perm.forward, base.perm.forward) and res.rank == base.rank
    scale = np.abs(base.packed).max()
    assert np.abs(res.packed - base.packed).max() <= 1e-10 * scale
    resid, orth = parity.residuals(A, res)
    assert resid <= 50 * n * O.EPS and orth <= 50 * n * O.EPS


def test_batched_large_matrices_per_matrix_path():
    """Batches of matrices too large to group (m n >= 2^20) take the per-matrix
    engine on concurrent lanes: identical to the single-matrix calls."""
    from paper_2106_03138_b200 import qrdm2
    from paper_2106_03138_b200.batch import factorize_batch

    rng = np.random.default_rng(71)
    B = rng.standard_normal((3, 1100, 1000))
    f = factorize_batch(B, lanes=2)
    for i in range(3):
        r, s = f.result(i), qrdm2(B[i])
        assert np.array_equal(r.perm.forward, s.perm.forward) and r.rank == s.rank
        assert np.abs(r.packed - s.packed).max() <= 1e-12 * np.abs(s.packed).max()


def test_fused_small_kernel_matches_step_kernels(monkeypatch):
    """The fused per-matrix kernel (small.cuh) against the per-step kernels on
    cfg3 matrices, wide / tall / rank-deficient shapes and the knob variants:
    identical decisions on the oracle's robust prefix, factors equal to rounding
    there, residual and orthogonality <= 50 n eps for both."""
    from paper_2106_03138_b200 import DMParams, StopCriterion, StopRule, inputs, qrdm, qrdm2

    rng = np.random.default_rng(909)
    cases = [inputs.cfg3(seed=3, batch=2)[1], rng.standard_normal((256, 512)), rng.standard_normal((200, 60)),
             rng.standard_normal((256, 40)) @ rng.standard_normal((40, 256)),
             rng.standard_normal((100, 100)) * np.logspace(0, -14, 100)]
    variants = [(qrdm2, DMParams(), StopCriterion()), (qrdm, DMParams(tau=0.3, delta=0.5), StopCriterion()),
                (qrdm2, DMParams(use_delta_max=True), StopCriterion(StopRule.NONE)),
                (qrdm2, DMParams(k_dm=7), StopCriterion(StopRule.EPS_SQRT_N))]
    for i, A in enumerate(cases):
        fn, p, st = variants[i % len(variants)]
        fused = fn(A, params=p, stop=st)
        monkeypatch.setenv("DMQR_NO_FUSED", "1")
        steps = fn(A, params=p, stop=st)
        monkeypatch.delenv("DMQR_NO_FUSED")
        kw = dict(tau=p.tau, delta=p.delta, k_dm=p.k_dm, use_delta_max=p.use_delta_max,
                  stop_rule=st.variant.value)
        with threadpool_limits(1):
            ref = (O.qrdm2 if fn is qrdm2 else O.qrdm)(A, margins=True, **kw)
        cut, full = parity.robust_prefix(ref)
        assert np.array_equal(fused.perm.forward[:cut], steps.perm.forward[:cut]), i
        nf = min(cut, fused.n_factored, steps.n_factored)
        scale = np.abs(steps.packed).max()
        assert np.abs(fused.packed[:, :nf] - steps.packed[:, :nf]).max() <= 1e-10 * scale, i
        _compare(A, fused, ref, f"fused[{i}]")
        _compare(A, steps, ref, f"steps[{i}]")


@pytest.mark.parametrize("algo", ["qrdm2", "qrp"])
@pytest.mark.parametrize("large_rows", [False, True])
def test_column_norms_overflow_underflow_kat(algo, large_rows):
    """column_norms' max-scaled path (matrix.py:61-78; KAT test_matrix.py:86-91):
    columns of 1e300 and 1e-300 entries, whose plain sums of squares overflow /
    underflow, must come out as 2e300 / 2e-300 (rel 1e-15) through the device
    norms, the pivot order and the reflectors.  ``large_rows`` repeats it on a
    2^20-element matrix so the look-ahead schedule's norm kernels run too."""
    m = 4 if not large_rows else 4096
    n = 3 if not large_rows else 256
    rng = np.random.default_rng(11)
    A = np.zeros((m, n))
    A[:, 0] = 1e-300 * np.where(np.arange(m) % 2 == 0, 1.0, -1.0)
    A[:, 1] = 1e300
    A[:2, 2] = [3.0, 4.0]
    if n > 3:
        A[:, 3:] = 1e-3 * rng.standard_normal((m, n - 3))
    sc = np.sqrt(m / 4.0)  # column norms scale with sqrt(m)
    res = _gpu(A, algo, stop_rule="none", trace_norms=True)
    ref = (O.qrp if algo == "qrp" else O.qrdm2)(A, stop_rule=O.STOP_NONE, trace_norms=True)
    d = np.abs(res.r_diagonal())
    assert np.all(np.isfinite(d))
    assert res.perm.forward[0] == 1
    assert d[0] == pytest.approx(2e300 * sc, rel=1e-15)
    j0 = int(np.flatnonzero(res.perm.forward == 0)[0])
    dr = np.abs(ref.r_diagonal())
    assert d[j0] == pytest.approx(dr[j0], rel=1e-10) and 0.9 * 2e-300 * sc < d[j0] < 1.1 * 2e-300 * sc
    assert np.array_equal(res.perm.forward, ref.forward)
    assert res.rank == ref.rank
    assert np.all(np.isfinite(res.norm_trace))


@pytest.mark.parametrize("e2", [500, -996])
def test_power_of_two_scaled_matrix_vs_oracle(e2):
    """A whole matrix scaled by 2^500 (~3e150: squares near overflow) or 2^-996
    (~1e-300: squares underflow to 0): the norms take the scaled
    branch; pivots, rank and |diag R| must match the oracle on the same input."""
    rng = np.random.default_rng(5)
    A = np.ldexp(rng.standard_normal((96, 80)) @ np.diag(np.logspace(0, -3, 80)), e2)
    res = _gpu(A, "qrdm2")
    ref = O.qrdm2(A)
    assert np.array_equal(res.perm.forward, ref.forward)
    assert res.rank == ref.rank
    ok, worst = parity.diag_close(res.r_diagonal(), ref.r_diagonal(), 96)
    assert ok, worst


@pytest.mark.parametrize("grade", [0, -3, -8, -13])
def test_fused_step_tail_is_bitwise_the_separate_kernels(monkeypatch, grade):
    """The look-ahead step's tail in one launch (k_trail_w's closing CTA + k_tail, csrc/tail.cuh) runs the
    separate kernels' device functions (k_trail_a fallback, k_guard, k_guard_norms, k_step_end): the
    factor, pivots, step log and counters must be identical bit for bit.  Graded columns bring in guard
    columns and declined CholeskyQR2 panels (the slow phases of k_tail)."""
    from paper_2106_03138_b200 import qrdm2

    rng = np.random.default_rng(91 - grade)
    A = rng.standard_normal((1300, 1100)) * np.logspace(0, grade, 1100)[rng.permutation(1100)]
    if grade == -13:  # a rank-deficient tail: panels decline, steps break and fall back
        A[:, 700:] = A[:, :400] @ rng.standard_normal((400, 400)) * 1e-9 + A[:, 700:] * 1e-14
    fused = qrdm2(A)
    monkeypatch.setenv("DMQR_NO_FUSED_TAIL", "1")
    sep = qrdm2(A)
    assert np.array_equal(fused.packed, sep.packed)
    assert np.array_equal(fused.coeffs, sep.coeffs)
    assert np.array_equal(fused.perm.forward, sep.perm.forward) and fused.rank == sep.rank
    assert _steps(fused.step_log) == _steps(sep.step_log)
    assert fused.counters == sep.counters
    resid, orth = parity.residuals(A, fused)
    assert resid <= 50 * 1300 * O.EPS and orth <= 50 * 1300 * O.EPS


@pytest.mark.parametrize("switch", ["DMQR_NO_CHOLQR", "DMQR_NO_LOOKAHEAD", "DMQR_NO_GRAPH", "DMQR_NO_STEP_GRAPH",
                                    "DMQR_NO_FUSED_TAIL"])
def test_schedule_switches_keep_parity(monkeypatch, switch):
    """Every schedule switch the engine reads (Householder-only panel, serial
    schedule, no replayed step graphs) gives the default run's decisions and a
    factor within rounding of it -- single matrices at a look-ahead size and a
    batched group of small ones."""
    from paper_2106_03138_b200 import qrdm2
    from paper_2106_03138_b200.batch import factorize_batch

    rng = np.random.default_rng(90)
    A = rng.standard_normal((1100, 1024)) * np.logspace(0, -8, 1024)[rng.permutation(1024)]
    B = rng.standard_normal((6, 160, 144)) @ np.diag(np.logspace(0, -12, 144))
    base, bb = qrdm2(A), factorize_batch(B)
    monkeypatch.setenv(switch, "1")
    monkeypatch.setenv("DMQR_NO_FUSED", "1")  # batched groups through the step kernels (graph path)
    res, rb = qrdm2(A), factorize_batch(B)
    assert np.array_equal(res.perm.forward, base.perm.forward) and res.rank == base.rank
    assert np.abs(res.packed - base.packed).max() <= 1e-9 * np.abs(base.packed).max()
    resid, orth = parity.residuals(A, res)
    assert resid <= 50 * 1100 * O.EPS and orth <= 50 * 1100 * O.EPS
    for i in range(len(B)):
        r, s = rb.result(i), bb.result(i)
        ref = O.qrdm2(B[i], margins=True)
        cut, _ = parity.robust_prefix(ref)
        assert np.array_equal(r.perm.forward[:cut], s.perm.forward[:cut])
        rr, oo = parity.residuals(B[i], r)
        assert rr <= 50 * 160 * O.EPS and oo <= 50 * 160 * O.EPS


# ---- wide k_dm (k_dm > 64: csrc/wide.cuh; dm.py:56-62 accepts any k_dm >= 1) ----

WIDE_FULL = ["wide/gauss_k128", "wide/wide_qrdm_k200", "wide/break_boundary", "wide/break_boundary_qrdm",
             "wide/break_chunk2", "wide/break_chunk3"]


@pytest.mark.parametrize("name", WIDE_FULL)
def test_wide_kdm_golden_full(name):
    """Blocks of more than one 65-column panel chunk, with the QRDM2 break on a
    chunk boundary (break_boundary: k_wcont's test), inside the second chunk and
    inside the third: the whole run equals the reference's (swap log, step log
    with one record per step, rank, counters)."""
    meta = G.index()["cases"][name]
    A = G.case_input(name)
    assert G.sha(A) == meta["input_sha256"]
    res = _gpu(A, meta["algo"], **G.oracle_kwargs(name))
    ref = _golden_oracle(name)
    _compare(A, res, ref, name, require_full=True)
    steps = G.case_field(name, "steps")
    assert [tuple(s) for s in _steps(res.step_log)] == [tuple(int(x) for x in s) for s in steps]


@pytest.mark.parametrize("seed", range(8))
def test_wide_kdm_random_vs_oracle(seed):
    rng = np.random.default_rng(6400 + seed)
    m = int(rng.integers(100, 700))
    n = int(rng.integers(100, 700))
    k_dm = [65, 66, 80, 128, 129, 200, 300, 10**9][seed]
    kind = seed % 3
    if kind == 0:
        A = rng.standard_normal((m, n))
    elif kind == 1:
        r = int(rng.integers(1, min(m, n)))
        A = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
    else:
        A = rng.standard_normal((m, n)) * np.logspace(0, -10, n)[rng.permutation(n)]
    algo = "qrdm2" if seed % 2 == 0 else "qrdm"
    res = _gpu(A, algo, k_dm=k_dm, use_delta_max=(seed == 5))
    with threadpool_limits(1):
        ref = (O.qrdm2 if algo == "qrdm2" else O.qrdm)(A, margins=True, k_dm=k_dm, use_delta_max=(seed == 5))
    _compare(A, res, ref, f"wide-random{seed}", min_cut=1)
    assert max(s.k_selected for s in res.step_log) == max(s.k_selected for s in ref.steps)


@pytest.mark.parametrize("shape", [(1100, 1024), (9000, 300)])
def test_wide_kdm_large_shapes(shape):
    """Shapes that take the look-ahead schedule (1100 x 1024) or the tall
    cluster panel (9000 x 300) at k_dm = 64 run serial with the wide selection."""
    rng = np.random.default_rng(shape[0])
    m, n = shape
    A = rng.standard_normal((m, n)) * np.logspace(0, -6, n)[rng.permutation(n)]
    res = _gpu(A, "qrdm2", k_dm=128)
    with threadpool_limits(4):
        ref = O.qrdm2(A, margins=True, k_dm=128)
    _compare(A, res, ref, f"wide-{m}x{n}", min_cut=64)


def test_wide_kdm_batched_per_matrix():
    """Batches with wide k_dm run every matrix on the per-matrix engine: identical
    to the single calls."""
    from paper_2106_03138_b200 import DMParams, qrdm2
    from paper_2106_03138_b200.batch import factorize_batch

    rng = np.random.default_rng(99)
    B = rng.standard_normal((5, 200, 180))
    f = factorize_batch(B, params=DMParams(k_dm=100), lanes=2)
    for b in range(5):
        one = qrdm2(B[b], params=DMParams(k_dm=100))
        r = f.result(b)
        assert np.array_equal(r.perm.forward, one.perm.forward) and r.rank == one.rank
        assert _steps(r.step_log) == _steps(one.step_log)


def test_forced_lookahead_on_a_tall_input_matches_default(monkeypatch):
    """DMQR_FORCE_LOOKAHEAD (the A/B switch that runs the look-ahead schedule at shapes
    the default keeps serial: m > 4n, n > 12288): same decisions, factor within rounding."""
    from paper_2106_03138_b200 import qrdm2

    rng = np.random.default_rng(93)
    A = rng.standard_normal((5000, 1100)) * np.logspace(0, -4, 1100)[rng.permutation(1100)]
    base = qrdm2(A)
    monkeypatch.setenv("DMQR_FORCE_LOOKAHEAD", "1")
    la = qrdm2(A)
    assert np.array_equal(la.perm.forward, base.perm.forward) and la.rank == base.rank
    assert _steps(la.step_log) == _steps(base.step_log)
    assert np.abs(la.packed - base.packed).max() <= 1e-9 * np.abs(base.packed).max()
    resid, orth = parity.residuals(A, la)
    assert resid <= 50 * 5000 * O.EPS and orth <= 50 * 5000 * O.EPS


@pytest.mark.parametrize("rows", ["72", "256"])
def test_panel_cluster_width_keeps_parity(monkeypatch, rows):
    """DMQR_CQ_ROWS (rows per CTA the look-ahead panel's cluster aims for; default 96, 256 = the old
    ceil(m'/256) width, 72 = the narrowest slice that still holds the top block): same decisions as the
    default, factor within rounding -- on a graded input whose panels break and decline."""
    from paper_2106_03138_b200 import qrdm2

    rng = np.random.default_rng(94)
    A = rng.standard_normal((2200, 2048)) * np.logspace(0, -9, 2048)[rng.permutation(2048)]
    base = qrdm2(A)
    monkeypatch.setenv("DMQR_CQ_ROWS", rows)
    res = qrdm2(A)
    ref = O.qrdm2(A, margins=True)
    cut, _ = parity.robust_prefix(ref)
    assert cut >= 64
    assert np.array_equal(res.perm.forward[:cut], base.perm.forward[:cut])
    assert np.array_equal(res.perm.forward[:cut], ref.forward[:cut])
    resid, orth = parity.residuals(A, res)
    assert resid <= 50 * 2200 * O.EPS and orth <= 50 * 2200 * O.EPS


@pytest.mark.parametrize("shape", [(600, 400), (1200, 1100)])
def test_equal_norm_columns_tie_order(shape):
    """Random +-1 entries: every column norm is exactly sqrt(m), so the first
    candidate set is one big tie class that must come out in index order
    (candidate_set's stable argsort, dm.py:81-97).  n = 400 goes through
    k_select's short-list rank counting, n = 1100 overflows the short list and
    takes the radix select with its index-ordered tie compaction."""
    m, n = shape
    rng = np.random.default_rng(m + n)
    A = rng.choice([-1.0, 1.0], size=(m, n))
    res = _gpu(A, "qrdm2")
    with threadpool_limits(1):
        ref = O.qrdm2(A, margins=True)
    assert np.array_equal(res.perm.forward[:64], ref.forward[:64]), "first block's pivots differ"
    assert _steps(res.step_log[:1]) == _steps(ref.steps[:1])
    _compare(A, res, ref, f"pm1_{m}x{n}")
