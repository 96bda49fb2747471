"""Which golden cases does the GPU reproduce exactly (whole perm, rank, step log)?
python tools/golden_exact.py  (GPU box)"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np  # noqa: E402

import golden_cases as G  # noqa: E402
from paper_2106_03138_b200 import DMParams, StopCriterion, StopRule, qrdm, qrdm2, qrp  # noqa: E402

exact, diff = [], []
for name in G.case_names():
    meta = G.index()["cases"][name]
    A = G.case_input(name)
    kw = G.oracle_kwargs(name)
    stop = StopCriterion(StopRule(kw["stop_rule"]))
    if meta["algo"] == "qrp":
        r = qrp(A, stop=stop)
    else:
        p = DMParams(tau=kw["tau"], delta=kw["delta"], k_dm=kw["k_dm"], use_delta_max=kw["use_delta_max"])
        r = (qrdm2 if meta["algo"] == "qrdm2" else qrdm)(A, params=p, stop=stop)
    f = G.case_field(name, "forward")
    ok = np.array_equal(r.perm.forward, f) and r.rank == meta["rank"] and r.n_factored == meta["n_factored"]
    if ok:
        exact.append(name)
    else:
        first = int(np.argmax(np.asarray(r.perm.forward) != f)) if not np.array_equal(r.perm.forward, f) else -1
        diff.append((name, first, r.rank, meta["rank"]))
print(f"exact {len(exact)} / {len(exact) + len(diff)}")
for d in diff:
    print("DIFF", d)
