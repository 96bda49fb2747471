"""Registry wiring (harness.py:40, 188-198 surface) -- host logic only, no GPU."""

import pytest

from paper_2106_03138_b200 import registry
from paper_2106_03138_b200.rrqr import DMParams, StopCriterion, StopRule


def test_same_names_as_reference_registry():
    assert set(registry.ALGORITHMS) == {"qrp", "qrdm", "qrdm2"}  # harness.py:40


def test_run_algorithm_dispatch(monkeypatch):
    calls = []
    for name in ("qrp", "qrdm", "qrdm2"):
        monkeypatch.setitem(registry.ALGORITHMS, name, lambda A, _n=name, **kw: calls.append((_n, sorted(kw))) or _n)
    p, st = DMParams(tau=0.2), StopCriterion(StopRule.NONE)
    assert registry.run_algorithm("qrp", None, p, st) == "qrp"
    assert registry.run_algorithm("qrdm2", None, p, st, trace_norms=True) == "qrdm2"
    assert calls == [("qrp", ["stop", "trace_norms"]), ("qrdm2", ["params", "stop", "trace_norms"])]
    with pytest.raises(KeyError):
        registry.run_algorithm("geqp3", None, p, st)


def test_register_into_reference_style_registry():
    ref = {"qrp": object(), "qrdm": object(), "qrdm2": object()}
    registry.register(ref)
    assert sorted(ref) == ["qrdm", "qrdm2", "qrdm2_b200", "qrdm_b200", "qrp", "qrp_b200"]
    # qrp_b200 accepts (and ignores) the params= keyword the reference passes to non-"qrp" names
    import inspect
    assert "params" in inspect.signature(ref["qrp_b200"]).parameters


def test_ratio_fields_identity_like_reference():
    """harness.py TestCompareRun.test_identity_all_algorithms: all ratios 1 on eye(8)."""
    import numpy as np
    from types import SimpleNamespace

    from paper_2106_03138_b200.diagnostics import ratio_fields

    res = SimpleNamespace(packed=np.eye(8), n_factored=8)
    out = ratio_fields(res, np.ones(8), 8, r11_svd="host")
    assert all(abs(v - 1.0) <= 1e-12 for v in out[:4]) and out[4] == ""
    short = ratio_fields(SimpleNamespace(packed=np.eye(8), n_factored=5), np.ones(8), 8, r11_svd="host")
    assert short[4] == "short_factorization"
