"""Where does the GPU first diverge from the oracle, and what were the oracle's
amplified margins there?  Calibrates the parity policy (run on the GPU box)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
from threadpoolctl import threadpool_limits

import golden_cases as G
from oracle import qrdm_oracle as O
from paper_2106_03138_b200 import DMParams, StopCriterion, StopRule, qrdm, qrdm2

rows = []
for name in G.case_names():
    meta = G.index()["cases"][name]
    A = G.case_input(name)
    kw = G.oracle_kwargs(name)
    with threadpool_limits(1):
        ref = (O.qrdm2 if meta["algo"] == "qrdm2" else O.qrdm)(A, margins=True, **kw)
    fn = qrdm2 if meta["algo"] == "qrdm2" else qrdm
    res = fn(A, params=DMParams(kw["tau"], kw["delta"], kw["k_dm"], kw["use_delta_max"]),
             stop=StopCriterion(StopRule(kw["stop_rule"])))
    nf = min(res.n_factored, ref.n_factored)
    diff = np.flatnonzero(res.perm.forward[:nf] != ref.forward[:nf])
    first = int(diff[0]) if diff.size else None
    same = first is None and res.rank == ref.rank and res.n_factored == ref.n_factored
    ps = ref.margins["per_step"]
    if first is not None:
        before = [g for (ns, g) in ps if ns <= first]
        at = min(before[-3:]) if before else None
        prior = min(before[:-1]) if len(before) > 1 else None
    else:
        at = prior = None
    rows.append((name, same, first, res.rank, ref.rank, ref.margins.get("first_ambiguous"), at, prior,
                 min(g for _, g in ps) if ps else None))
    print(f"{name:45s} same={same!s:5} first_div={first} rank gpu/ref={res.rank}/{ref.rank} "
          f"first_amb={ref.margins.get('first_ambiguous')} amp_at_div={at} min_amp_all={rows[-1][-1]}",
          flush=True)
