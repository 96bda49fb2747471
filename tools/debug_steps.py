"""Step-by-step GPU vs oracle comparison (debug aid; run on the GPU box)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from oracle import qrdm_oracle as O
from paper_2106_03138_b200 import rrqr


def run(A, steps, **kw):
    f = rrqr.factorize(A, max_steps=steps, **kw)
    d = f.debug_ctl()
    print("   ctl:", {k: v for k, v in d.items() if not isinstance(v, list)})
    print("   cand:", d["cand"][:d["ncand"]], "sel:", d["sel"][:d["nsel"]])
    return rrqr.to_result(f)


def compare(label, A, nsteps=3, **kw):
    print(f"=== {label} {A.shape}")
    for s in range(1, nsteps + 1):
        g = run(A, s)
        o = O.qrdm2(A, max_steps=s)
        sd, cd = O.candidates(O.col_norms(A), 0.15, 64)
        print("   oracle seed/cand (step1):", sd, cd[:12])
        gs = [(x.n_s, x.k_selected, x.k_accepted, x.k_max, x.broke_early) for x in g.step_log]
        os_ = [(x.n_s, x.k_selected, x.k_accepted, x.k_max, x.broke_early) for x in o.steps]
        print(f" step {s}: gpu {gs[-1:]}  ora {os_[-1:]}")
        print(f"   perm equal: {np.array_equal(g.perm.forward, o.forward)}  swaps gpu[:6]={g.perm.swaps[:6]} ora[:6]={o.swaps[:6]}")
        dp = np.abs(g.packed - o.packed)
        print(f"   packed max diff {dp.max():.3e} at {np.unravel_index(dp.argmax(), dp.shape)}; coeffs diff {np.abs(g.coeffs - o.coeffs).max():.3e}")
        nf = o.n_factored
        print(f"   diag gpu {g.packed.diagonal()[:4]} ora {o.packed.diagonal()[:4]}")
        if dp.max() > 1e-8:
            # which region differs
            ns = o.steps[-1].n_s if o.steps else 0
            reg = {
                "R rows/cols<n_s1": dp[:nf, :].max() if nf else 0,
                "panel cols": dp[:, ns:nf].max() if nf > ns else 0,
                "trailing": dp[nf:, nf:].max() if nf < min(A.shape) else 0,
            }
            print("   region diffs:", {k: f"{v:.2e}" for k, v in reg.items()})
            return


if __name__ == "__main__":
    rng = np.random.default_rng(0)
    compare("tiny 12x10", rng.standard_normal((12, 10)), 2)
    compare("small 40x30", rng.standard_normal((40, 30)), 2)
    compare("300x200", rng.standard_normal((300, 200)), 3)
    compare("600x500", rng.standard_normal((600, 500)), 3)
