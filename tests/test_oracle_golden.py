"""Pin the CPU oracle (oracle/qrdm_oracle.py) to the reference's own outputs.

Golden vectors come from running the reference dmqr package itself
(tests/golden/make_golden.py).  The oracle restates the same numpy operation
sequence, so with one BLAS thread it must agree BIT FOR BIT.  CPU only.
"""

import numpy as np
import pytest
from threadpoolctl import threadpool_limits

import golden_cases as G
from oracle import qrdm_oracle as O

CASES = [c for c in G.case_names() if not c.startswith(("cfg4s", "cfg2s"))]
SLOW = [c for c in G.case_names() if c.startswith(("cfg4s", "cfg2s"))]


def _check(name):
    meta = G.index()["cases"][name]
    A = G.case_input(name)
    assert G.sha(A) == meta["input_sha256"], "input generator does not reproduce the reference input"
    with threadpool_limits(1):
        if meta["algo"] == "qrp":
            res = O.qrp(A, stop_rule=meta["stop"])
        else:
            fn = O.qrdm2 if meta["algo"] == "qrdm2" else O.qrdm
            res = fn(A, **G.oracle_kwargs(name))
    f = lambda k: G.case_field(name, k)  # noqa: E731
    assert np.array_equal(res.forward, f("forward"))
    assert np.array_equal(np.array(res.swaps, dtype=np.int64).reshape(-1, 2), f("swaps"))
    assert res.rank == int(f("rank"))
    assert res.n_factored == int(f("n_factored"))
    assert int(res.stopped_early) == int(f("stopped_early"))
    assert np.array_equal(res.r_diagonal(), f("diag"))
    assert np.array_equal(res.coeffs, f("coeffs"))
    steps = np.array([[s.n_s, s.k_selected, s.k_accepted, int(s.broke_early),
                       int(s.fell_back_to_scalar),
                       -1 if (s.fell_back_to_scalar or meta["algo"] == "qrp") else s.k_max]
                      for s in res.steps], dtype=np.int64).reshape(-1, 6)
    assert np.array_equal(steps, f("steps"))
    eg = np.array([[s.eps_s, s.gamma] for s in res.steps]).reshape(-1, 2)
    assert np.array_equal(eg, f("eps_gamma"))
    assert np.array_equal(np.array(res.counters), f("counters"))
    if meta["packed"]:
        assert np.array_equal(res.packed, f("packed"))


@pytest.mark.parametrize("name", CASES)
def test_oracle_bit_exact_vs_reference(name):
    _check(name)


@pytest.mark.slow
@pytest.mark.parametrize("name", SLOW)
def test_oracle_bit_exact_vs_reference_midsize(name):
    _check(name)


def test_fixture_count_is_40():
    import fixture_suite
    assert len(fixture_suite.suite()) == 40


def test_qrp_cases_present():
    names = G.case_names("qrp/")
    assert len(names) >= 50
    assert any(G.index()["cases"][c]["stop"] == "none" for c in names)


def test_cfg1_rank_384():
    assert G.index()["cases"]["cfg1/qrdm2"]["rank"] == 384
    assert G.index()["cases"]["cfg1/qrdm"]["rank"] == 390
