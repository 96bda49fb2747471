"""Full-size golden summaries for the BASELINE configs, made by running the REFERENCE.

Run here (the build container), where /root/reference exists:

    python tests/golden/make_fullsize.py [cfg3] [cfg4] [cfg5_4096] [cfg5_8192] [cfg5_16384]

For each case it generates the BASELINE input on the host with one OpenBLAS
thread (``paper_2106_03138_b200.inputs``, byte-reproducible; its sha256 is
stored), runs the reference ``dmqr.qrdm2`` (rrqr.py:443-456) with the default
``DMParams()`` / ``StopCriterion()``, and runs the oracle port on the same input
with its margin trace so the GPU tests know which decisions are
robust.  The oracle must reproduce the reference exactly (it is pinned bit for
bit on the small cases, ``tests/test_oracle_golden.py``); the script asserts
that here too.  Stored per case (``fullsize.npz`` + ``fullsize_index.json``):
input sha256, forward permutation, rank, n_factored, stopped_early, |diag R|,
coeffs, step log (n_s, k_sel, k_acc, broke, fallback, k_max), eps_s / gamma,
analytic counters, and the oracle's first-ambiguous column and per-step
minimum scaled margins.  Nothing on the GPU box reads /root/reference.

cfg3 (1024 matrices) runs one matrix per worker process (``multiprocessing``,
one BLAS thread each: the drivers are pure functions, README.md:146-147).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

os.environ["OPENBLAS_NUM_THREADS"] = "1"
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")

import numpy as np  # noqa: E402

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

OUT_NPZ = HERE / "fullsize.npz"
OUT_IDX = HERE / "fullsize_index.json"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.float64)).tobytes(order="C")).hexdigest()


def summarize(A: np.ndarray) -> dict:
    """Reference qrdm2 + oracle margins on one input -> compact summary."""
    import dmqr.rrqr as R
    from dmqr.dm import DMParams
    from dmqr.rrqr import StopCriterion

    from oracle import qrdm_oracle as O

    kmax_log: list = []
    orig = R.dm_select

    def traced(*a, **kw):  # k_max of every DM step (SURVEY App. D hook, rrqr.py:340)
        sel = orig(*a, **kw)
        kmax_log.append(sel.k_max)
        return sel

    R.dm_select = traced
    try:
        t0 = time.perf_counter()
        res = R.qrdm2(A, params=DMParams(), stop=StopCriterion())
        t_ref = time.perf_counter() - t0
    finally:
        R.dm_select = orig
    it = iter(kmax_log)
    steps = np.array([[s.n_s, s.k_selected, s.k_accepted, int(s.broke_early), int(s.fell_back_to_scalar),
                       -1 if s.fell_back_to_scalar else next(it)] for s in res.step_log],
                     dtype=np.int64).reshape(-1, 6)
    t0 = time.perf_counter()
    orc = O.qrdm2(A, margins=True)
    t_orc = time.perf_counter() - t0
    same = (np.array_equal(orc.forward, res.perm.forward) and orc.rank == res.rank
            and np.array_equal(orc.r_diagonal(), res.r_diagonal()))
    fa = orc.margins.get("first_ambiguous")
    per_step = np.array(orc.margins.get("per_step", []), dtype=np.float64).reshape(-1, 2)
    c = res.counters
    return dict(
        sha=sha(A), t_ref=t_ref, t_orc=t_orc, oracle_equal=bool(same),
        first_ambiguous=-1 if fa is None else int(fa),
        forward=np.asarray(res.perm.forward, dtype=np.int32),
        rank=int(res.rank), n_factored=int(res.n_factored), stopped_early=int(res.stopped_early),
        diag=np.asarray(res.r_diagonal(), dtype=np.float64),
        coeffs=np.asarray(res.coeffs, dtype=np.float64),
        steps=steps,
        eps_gamma=np.array([[s.eps_s, s.gamma] for s in res.step_log], dtype=np.float64).reshape(-1, 2),
        counters=np.array([c.rank1_flops, c.blocked_flops, c.total_flops]),
        margins=per_step,
        n_swaps=len(res.perm.swaps),
    )


def _cfg3_one(b: int) -> dict:
    from paper_2106_03138_b200 import inputs

    A = _CFG3[b]
    return summarize(A)


_CFG3 = None


def _cfg3_init():
    global _CFG3
    from paper_2106_03138_b200 import inputs

    _CFG3 = inputs.cfg3(seed=3, batch=1024)


def load_existing():
    store, index = {}, {"cases": {}}
    if OUT_NPZ.exists():
        with np.load(OUT_NPZ) as z:
            store = {k: z[k] for k in z.files}
    if OUT_IDX.exists():
        index = json.loads(OUT_IDX.read_text())
    return store, index


def save(store, index):
    import dmqr

    index.update({"numpy": np.__version__, "openblas_threads": 1, "reference": "dmqr " + dmqr.__version__})
    np.savez_compressed(OUT_NPZ, **store)
    OUT_IDX.write_text(json.dumps(index, indent=1, sort_keys=True))


SCALARS = ("rank", "n_factored", "stopped_early", "first_ambiguous", "n_swaps")
ARRAYS = ("forward", "diag", "coeffs", "steps", "eps_gamma", "counters", "margins")


def put(store, index, case, s, meta):
    for k in ARRAYS:
        store[f"{case}/{k}"] = s[k]
    index["cases"][case] = dict(meta, input_sha256=s["sha"], t_ref_s=round(s["t_ref"], 3),
                                t_oracle_s=round(s["t_orc"], 3), oracle_equal=s["oracle_equal"],
                                **{k: s[k] for k in SCALARS})
    print(f"{case:24s} rank={s['rank']:6d} steps={len(s['steps']):5d} first_amb={s['first_ambiguous']:6d} "
          f"ref {s['t_ref']:.1f}s oracle {s['t_orc']:.1f}s equal={s['oracle_equal']}", flush=True)


def main(which):
    from paper_2106_03138_b200 import inputs

    store, index = load_existing()
    if "cfg4" in which:
        A = inputs.cfg4(seed=4)
        put(store, index, "cfg4", summarize(A), dict(m=65536, n=1024, source="inputs.cfg4(seed=4)"))
        save(store, index)
        del A
    for n in (4096, 8192, 16384):  # (16384: ~45 min each for the reference and the oracle, one thread)
        if f"cfg5_{n}" in which:
            A = inputs.cfg5(seed=4, n=n)
            put(store, index, f"cfg5_{n}", summarize(A), dict(m=n, n=n, source=f"inputs.cfg5(seed=4,n={n})"))
            save(store, index)
            del A
    if "cfg3" in which:
        import multiprocessing as mp

        with mp.get_context("fork").Pool(os.cpu_count(), initializer=_cfg3_init) as pool:
            outs = pool.map(_cfg3_one, range(1024), chunksize=8)
        B = inputs.cfg3(seed=3, batch=1024)
        sh = [sha(B[b]) for b in range(1024)]
        assert all(o["sha"] == h for o, h in zip(outs, sh))
        # per-matrix arrays stacked (all matrices are 256 x 256)
        store["cfg3/forward"] = np.stack([o["forward"] for o in outs]).astype(np.int16)
        store["cfg3/diag"] = np.stack([np.pad(o["diag"], (0, 256 - o["diag"].size)) for o in outs])
        store["cfg3/rank"] = np.array([o["rank"] for o in outs], dtype=np.int32)
        store["cfg3/n_factored"] = np.array([o["n_factored"] for o in outs], dtype=np.int32)
        store["cfg3/first_ambiguous"] = np.array([o["first_ambiguous"] for o in outs], dtype=np.int32)
        store["cfg3/n_steps"] = np.array([len(o["steps"]) for o in outs], dtype=np.int32)
        store["cfg3/steps"] = np.concatenate([o["steps"] for o in outs])
        store["cfg3/eps_s"] = np.concatenate([o["eps_gamma"][:, 0] for o in outs])
        store["cfg3/counters"] = np.stack([o["counters"] for o in outs])
        index["cases"]["cfg3"] = dict(
            m=256, n=256, batch=1024, source="inputs.cfg3(seed=3,batch=1024)",
            input_sha256=hashlib.sha256("".join(sh).encode()).hexdigest(),
            oracle_equal=all(o["oracle_equal"] for o in outs),
            t_ref_s=round(sum(o["t_ref"] for o in outs), 2),
            rank_histogram={str(r): int(c) for r, c in zip(*np.unique(store["cfg3/rank"], return_counts=True))})
        print("cfg3 ranks", index["cases"]["cfg3"]["rank_histogram"], "oracle_equal",
              index["cases"]["cfg3"]["oracle_equal"], flush=True)
        save(store, index)


if __name__ == "__main__":
    main(set(sys.argv[1:]) or {"cfg3", "cfg4", "cfg5_4096"})
