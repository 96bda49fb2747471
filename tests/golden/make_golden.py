"""Generate golden vectors by running the REFERENCE implementation itself.

Run here (the build container), where /root/reference exists:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

It imports the reference package ``dmqr`` (read-only tree at
/root/reference/pkg/src; numba cache redirected to /tmp), feeds it the inputs
below, and stores the public result fields of ``qrdm`` / ``qrdm2``
(rrqr.py:136-158) plus the candidate-set size k_max (traced through the
module-global ``dm_select`` hook) in ``golden.npz`` with a JSON
index.  Nothing on the GPU box reads /root/reference; the committed outputs
are the pin for ``oracle/qrdm_oracle.py`` and for the GPU parity tests.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")

import numpy as np  # noqa: E402

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tests"))

import dmqr  # noqa: E402
import dmqr.rrqr as R  # noqa: E402
from dmqr.dm import DMParams  # noqa: E402
from dmqr.rrqr import StopCriterion, StopRule  # noqa: E402

from paper_2106_03138_b200 import inputs  # noqa: E402

# capture k_max of every DM step via the module-global hook (rrqr.py:340)
_KMAX: list = []
_orig_select = R.dm_select


def _traced_select(*a, **kw):
    sel = _orig_select(*a, **kw)
    _KMAX.append(sel.k_max)
    return sel


R.dm_select = _traced_select


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.float64)).tobytes(order="C")).hexdigest()


def run_ref(A, algo, params, stop):
    _KMAX.clear()
    if algo == "qrp":  # rrqr.py:238-291 (no DM selection, no params)
        res = R.qrp(A, stop=stop)
    else:
        fn = R.qrdm2 if algo == "qrdm2" else R.qrdm
        res = fn(A, params=params, stop=stop)
    kmax_iter = iter(list(_KMAX))
    steps = []
    for rec in res.step_log:
        km = -1 if (rec.fell_back_to_scalar or algo == "qrp") else next(kmax_iter)
        steps.append([rec.n_s, rec.k_selected, rec.k_accepted, int(rec.broke_early),
                      int(rec.fell_back_to_scalar), km])
    steps = np.array(steps, dtype=np.int64).reshape(-1, 6)
    eps_gamma = np.array([[rec.eps_s, rec.gamma] for rec in res.step_log], dtype=np.float64).reshape(-1, 2)
    sw = np.array(res.perm.swaps, dtype=np.int64).reshape(-1, 2)
    c = res.counters
    return dict(
        forward=np.asarray(res.perm.forward, dtype=np.int64),
        swaps=sw,
        rank=np.int64(res.rank),
        n_factored=np.int64(res.n_factored),
        stopped_early=np.int64(res.stopped_early),
        diag=res.r_diagonal(),
        coeffs=np.asarray(res.coeffs),
        steps=steps,
        eps_gamma=eps_gamma,
        counters=np.array([c.rank1_flops, c.blocked_flops, c.total_flops]),
        packed=np.asarray(res.packed),
    )


def main():
    store: dict = {}
    index: dict = {"numpy": np.__version__, "openblas_threads": os.environ["OPENBLAS_NUM_THREADS"],
                   "reference": "dmqr " + dmqr.__version__, "cases": {}}

    def add(case, A, algo, params, stop, source, keep_packed=False, keep_input=False):
        out = run_ref(A, algo, params, stop)
        meta = dict(m=int(A.shape[0]), n=int(A.shape[1]), algo=algo, tau=params.tau,
                    delta=params.delta, k_dm=params.k_dm, use_delta_max=params.use_delta_max,
                    stop=stop.variant.value, source=source, input_sha256=sha(A),
                    rank=int(out["rank"]), n_factored=int(out["n_factored"]),
                    packed=keep_packed, input=keep_input)
        for k, v in out.items():
            if k == "packed" and not keep_packed:
                continue
            store[f"{case}/{k}"] = v
        if keep_input:
            store[f"{case}/input"] = np.asarray(A, dtype=np.float64)
        index["cases"][case] = meta
        print(f"{case:48s} {algo:6s} rank={meta['rank']:5d} steps={len(out['steps'])}")

    D = DMParams()
    EPSN = StopCriterion()
    NONE = StopCriterion(StopRule.NONE)
    SQRT = StopCriterion(StopRule.EPS_SQRT_N)

    # 1. the reference's own 40-matrix fixture suite (harness.py:135-185)
    for i, (name, A) in enumerate(dmqr.fixture_suite()):
        small = A.shape[0] * A.shape[1] <= 96 * 96
        add(f"fix/{name}/qrdm2", A, "qrdm2", D, EPSN, "fixture", keep_packed=small and i % 3 == 0)
        add(f"fix/{name}/qrdm", A, "qrdm", D, EPSN, "fixture")
        add(f"fix/{name}/qrdm2_none", A, "qrdm2", D, NONE, "fixture")

    # 2. BASELINE cfg1 (512^2, numerical rank 384) -- the PR1 oracle check
    A1 = inputs.cfg1(seed=0)
    add("cfg1/qrdm2", A1, "qrdm2", D, EPSN, "inputs.cfg1(seed=0)")
    add("cfg1/qrdm", A1, "qrdm", D, EPSN, "inputs.cfg1(seed=0)")
    add("cfg1/qrdm2_none", A1, "qrdm2", D, NONE, "inputs.cfg1(seed=0)")

    # 3. scaled-down stand-ins of cfg2..cfg5 (same recipes, sizes the CPU finishes fast)
    add("cfg2s/1024", inputs.cfg2(seed=1, n=1024), "qrdm2", D, EPSN, "inputs.cfg2(seed=1,n=1024)")
    B3 = inputs.cfg3(seed=3, batch=4)
    for b in range(4):
        add(f"cfg3s/{b}", B3[b], "qrdm2", D, EPSN, f"inputs.cfg3(seed=3,batch=4)[{b}]")
    add("cfg4s/8192x256", inputs.cfg4(seed=4, m=8192, n=256), "qrdm2", D, EPSN,
        "inputs.cfg4(seed=4,m=8192,n=256)")
    add("cfg5s/1024", inputs.cfg5(seed=4, n=1024), "qrdm2", D, EPSN, "inputs.cfg5(seed=4,n=1024)")

    # 4. knob coverage on small random inputs (stored with their inputs)
    rng = np.random.default_rng(2106)
    for t in range(24):
        m = int(rng.integers(2, 80))
        n = int(rng.integers(2, 80))
        kind = t % 3
        if kind == 0:
            A = rng.standard_normal((m, n))
        elif kind == 1:
            r = int(rng.integers(1, min(m, n) + 1))
            A = rng.standard_normal((m, r)) @ rng.standard_normal((r, n))
        else:
            A = rng.standard_normal((m, n)) * np.logspace(0, -12, n)
        kdm = int(rng.integers(1, 12))
        variants = [
            ("qrdm2", DMParams(k_dm=kdm), NONE),
            ("qrdm", DMParams(tau=0.3, delta=0.5), SQRT),
            ("qrdm2", DMParams(use_delta_max=True), EPSN),
            ("qrdm", DMParams(delta=0.0), NONE),
        ]
        algo, p, st = variants[t % 4]
        add(f"knob/{t}", A, algo, p, st, "make_golden rng(2106)", keep_packed=True, keep_input=True)

    # 5. reference KATs re-targeted (test_rrqr.py:78-149,299-320)
    add("kat/identity4", np.eye(4), "qrdm", DMParams(tau=0.5, delta=0.5, k_dm=8), EPSN, "eye(4)",
        keep_packed=True, keep_input=True)
    r33 = np.random.default_rng(33)
    a, b = r33.standard_normal(8), r33.standard_normal(8)
    add("kat/duplicate", np.column_stack([a, a, b]), "qrdm", DMParams(tau=0.1, delta=0.9), EPSN,
        "test_rrqr.py:84-94", keep_packed=True, keep_input=True)
    r38 = np.random.default_rng(38)
    q = np.linalg.qr(r38.standard_normal((20, 20)))
    q = q[0] * np.sign(np.diagonal(q[1]))
    Abrk = np.column_stack([q[:, 0], 0.98 * q[:, 1] + 0.05 * q[:, 0],
                            0.95 * (0.6 * q[:, 0] + 0.79 * q[:, 1]) + 0.01 * q[:, 2],
                            0.90 * q[:, 2] + 0.02 * q[:, 0]])
    add("kat/break", Abrk, "qrdm2", DMParams(tau=0.15, delta=0.95, k_dm=8), NONE,
        "test_rrqr.py:136-149", keep_packed=True, keep_input=True)
    r46 = np.random.default_rng(46)
    for (m, n) in [(5, 20), (20, 5), (1, 7), (7, 1)]:
        A = r46.standard_normal((m, n))
        add(f"kat/shape_{m}x{n}", A, "qrdm2", D, NONE, "test_rrqr.py:311-320",
            keep_packed=True, keep_input=True)
    add("kat/zeros", np.zeros((4, 3)), "qrdm2", D, EPSN, "zeros", keep_packed=True, keep_input=True)
    r36 = np.random.default_rng(36)
    A = r36.standard_normal((12, 4)) @ r36.standard_normal((4, 10))
    add("kat/fallback", A, "qrdm", D, NONE, "test_rrqr.py:118-123", keep_packed=True, keep_input=True)

    # 6. qrp (greedy column pivoting, rrqr.py:238-291): the blocked scalar-pivot
    #    engine's pins (it also runs QRDM's scalar-fallback runs)
    for i, (name, A) in enumerate(dmqr.fixture_suite()):
        add(f"qrp/fix/{name}", A, "qrp", D, EPSN if i % 2 == 0 else NONE, "fixture",
            keep_packed=A.shape[0] * A.shape[1] <= 96 * 96 and i % 3 == 0)
    add("qrp/cfg1", A1, "qrp", D, EPSN, "inputs.cfg1(seed=0)")
    add("qrp/cfg1_none", A1, "qrp", D, NONE, "inputs.cfg1(seed=0)")
    add("qrp/cfg5s/1024", inputs.cfg5(seed=4, n=1024), "qrp", D, EPSN, "inputs.cfg5(seed=4,n=1024)")
    rq = np.random.default_rng(238)
    for t in range(12):
        m = int(rq.integers(1, 100))
        n = int(rq.integers(1, 100))
        if t % 3 == 0:
            A = rq.standard_normal((m, n))
        elif t % 3 == 1:
            r = int(rq.integers(1, min(m, n) + 1))
            A = rq.standard_normal((m, r)) @ rq.standard_normal((r, n))
        else:
            A = rq.standard_normal((m, n)) * np.logspace(0, -14, n)
        st = (EPSN, SQRT, NONE)[t % 3]
        add(f"qrp/knob/{t}", A, "qrp", D, st, "make_golden rng(238)", keep_packed=True, keep_input=True)
    add("qrp/kat/zeros", np.zeros((5, 4)), "qrp", D, EPSN, "zeros", keep_packed=True, keep_input=True)
    add("qrp/kat/identity6", np.eye(6), "qrp", D, NONE, "eye(6)", keep_packed=True, keep_input=True)

    np.savez_compressed(HERE / "golden.npz", **store)
    (HERE / "golden_index.json").write_text(json.dumps(index, indent=1, sort_keys=True))
    print("cases:", len(index["cases"]), "bytes:", (HERE / "golden.npz").stat().st_size)


if __name__ == "__main__":
    main()
