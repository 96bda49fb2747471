"""Add the wide-k_dm golden cases (k_dm > 64, tests/wide_cases.py) to
golden.npz / golden_index.json by running the REFERENCE itself (same capture
as make_golden.py, whose run_ref this reuses).  Run here, where
/root/reference exists:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_wide.py

Inputs are not stored: the tests regenerate them from the seeded recipes and
check the recorded sha256.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
import make_golden as MG  # noqa: E402  (imports the reference, installs the k_max hook)
import wide_cases as WC  # noqa: E402  (tests/ is on sys.path via make_golden)


def main():
    store = dict(np.load(HERE / "golden.npz"))
    index = json.loads((HERE / "golden_index.json").read_text())
    stops = {"eps*n": MG.StopCriterion(), "none": MG.StopCriterion(MG.StopRule.NONE)}
    for case, inp, algo, k_dm, extra, stop in WC.CASES:
        A = WC.make(inp)
        params = MG.DMParams(k_dm=k_dm, **extra)
        out = MG.run_ref(A, algo, params, stops[stop])
        for k in [k for k in store if k.startswith(case + "/")]:
            del store[k]
        for k, v in out.items():
            if k != "packed":
                store[f"{case}/{k}"] = v
        index["cases"][case] = dict(
            m=int(A.shape[0]), n=int(A.shape[1]), algo=algo, tau=params.tau, delta=params.delta,
            k_dm=params.k_dm, use_delta_max=params.use_delta_max, stop=stops[stop].variant.value,
            source=f"wide:{inp}", input_sha256=MG.sha(A), rank=int(out["rank"]),
            n_factored=int(out["n_factored"]), packed=False, input=False)
        st = out["steps"]
        print(f"{case:32s} rank={int(out['rank']):4d} steps={len(st)} max k_s={st[:, 1].max()} "
              f"broke={int(st[:, 3].sum())}")
    np.savez_compressed(HERE / "golden.npz", **store)
    (HERE / "golden_index.json").write_text(json.dumps(index, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
