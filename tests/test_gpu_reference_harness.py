"""The reference's own harness and CLI driving the B200 engine.

`registry.register` adds ``qrp_b200`` / ``qrdm_b200`` / ``qrdm2_b200`` to the
reference's ``ALGORITHMS`` (harness.py:40); then the unmodified
``compare_run`` (harness.py:219-272), ``rows_to_csv`` (harness.py:283-307) and
``dmqr factor|compare --algo`` (cli.py:46, 102-137) run them next to the
reference's CPU drivers.  The reference comes from the pip install in
baseline/_ref (it travels with the repo snapshot); without it these tests skip.
"""

from __future__ import annotations

import csv
import io
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dmqr():
    if not (REF / "dmqr").is_dir():
        pytest.skip("reference package not installed in baseline/_ref (see DESIGN.md §5)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/dmqr_numba_cache")
    sys.path.insert(0, str(REF))
    try:
        import dmqr as mod
        import dmqr.cli  # noqa: F401
        import dmqr.harness  # noqa: F401
    finally:
        sys.path.remove(str(REF))
    from paper_2106_03138_b200 import registry

    saved = dict(mod.harness.ALGORITHMS)
    registry.register(mod.harness.ALGORITHMS)
    yield mod
    mod.harness.ALGORITHMS.clear()
    mod.harness.ALGORITHMS.update(saved)


def _suite(dmqr, names):
    suite = dict(dmqr.harness.fixture_suite())
    return [(nm, suite[nm]) for nm in names]


CASES = ["cliff_m96_n64_r48_g1e+04", "cliff_m128_n128_r112_g1e+04", "fullrank_m128_n128_k1e+06"]


def test_compare_run_with_b200_algorithms(dmqr):
    mats = _suite(dmqr, CASES)
    algos = ["qrp", "qrp_b200", "qrdm", "qrdm_b200", "qrdm2", "qrdm2_b200"]
    rows = dmqr.harness.compare_run(mats, algos)
    assert len(rows) == len(mats) * len(algos)
    by = {(r.matrix, r.algo): r for r in rows}
    for name, _ in mats:
        for a in ("qrp", "qrdm", "qrdm2"):
            ref, dev = by[(name, a)], by[(name, a + "_b200")]
            assert dev.rank_computed == ref.rank_computed, (name, a)
            assert dev.rank_oracle == ref.rank_oracle
            assert dev.breaks == ref.breaks and dev.fallbacks == ref.fallbacks, (name, a)
            assert dev.mean_ks == pytest.approx(ref.mean_ks), (name, a)
            for f in ("ratio_d_min", "ratio_d_max", "ratio_s_min", "ratio_s_max"):
                assert getattr(dev, f) == pytest.approx(getattr(ref, f), rel=1e-8), (name, a, f)
            assert dev.flags == ref.flags
    text = dmqr.harness.rows_to_csv(rows)
    parsed = list(csv.reader(io.StringIO(text)))
    assert len(parsed) == 1 + len(rows)
    assert {r[1] for r in parsed[1:]} == set(algos)


def test_cli_factor_and_compare(dmqr, tmp_path, capsys):
    from dmqr.mmio import write_matrix_market

    name, A = _suite(dmqr, ["cliff_m96_n96_r72_g1e+04"])[0]
    path = tmp_path / f"{name}.mtx"
    write_matrix_market(path, A)
    outs = {}
    for algo in ("qrdm2", "qrdm2_b200"):
        out = tmp_path / f"factor_{algo}.txt"
        assert dmqr.cli.main(["factor", "--input", str(path), "--algo", algo, "--out", str(out)]) == 0
        outs[algo] = out.read_text().splitlines()
    # same rank / factored count / step summary / leading pivots; only the algo line and time differ
    for i in (0, 3, 4):
        assert outs["qrdm2"][i] == outs["qrdm2_b200"][i]
    rank_line = lambda s: s.split("time_s")[0]  # noqa: E731
    assert rank_line(outs["qrdm2"][2]) == rank_line(outs["qrdm2_b200"][2])
    csv_out = tmp_path / "cmp.csv"
    rc = dmqr.cli.main(["compare", "--inputs", str(path), "--algos", "qrdm2,qrdm2_b200", "--out", str(csv_out)])
    assert rc == 0
    rows = list(csv.reader(io.StringIO(csv_out.read_text())))
    assert [r[1] for r in rows[1:]] == ["qrdm2", "qrdm2_b200"]
    assert rows[1][5] == rows[2][5]  # rank_computed
    # unknown names still fail the reference's way (exit code 1)
    with pytest.raises(SystemExit) as ei:
        dmqr.cli.main(["compare", "--inputs", str(path), "--algos", "geqp3_b200"])
    assert ei.value.code == 1


def test_reference_param_objects_accepted(dmqr):
    """The harness passes the reference's own DMParams / StopCriterion objects."""
    from paper_2106_03138_b200 import qrdm2

    A = _suite(dmqr, ["cliff_m64_n48_r32_g1e+04"])[0][1]
    for rule in ("n", "sqrt-n", "none"):
        st = dmqr.rrqr.StopCriterion.from_name(rule)
        p = dmqr.dm.DMParams(tau=0.2, delta=0.8)
        ref = dmqr.qrdm2(A, params=p, stop=st)
        dev = qrdm2(A, params=p, stop=st)
        assert dev.rank == ref.rank
        assert np.array_equal(dev.perm.forward, ref.perm.forward)
