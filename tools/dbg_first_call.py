import sys, os
sys.path[:0] = [__import__('os').environ.get('PKGROOT', '/root/repo'), '/root/repo', '/root/repo/tests']
import numpy as np
import golden_cases as G
from paper_2106_03138_b200 import qrdm, qrdm2, inputs, DMParams
name = "cfg1/qrdm"
A = G.case_input(name)
f = G.case_field(name, "forward")
for i in range(3):
    r = qrdm(A)
    d = np.flatnonzero(r.perm.forward != f)
    print(i, "rank", r.rank, "first diff", d[:5], "nsteps", len(r.step_log), [(s.n_s, s.k_selected, s.k_accepted) for s in r.step_log][:8], flush=True)
# random4 / random9 of test_random_vs_oracle (fused)
for seed in (4, 9, 1, 2):
    rng = np.random.default_rng(1000 + seed)
    m = int(rng.integers(40, 400)); n = int(rng.integers(40, 400))
    kind = seed % 3
    if kind == 0: A = rng.standard_normal((m, n))
    elif kind == 1:
        rr = int(rng.integers(1, min(m, n))); A = rng.standard_normal((m, rr)) @ rng.standard_normal((rr, n))
    else: A = rng.standard_normal((m, n)) * np.logspace(0, -10, n)[rng.permutation(n)]
    fn = qrdm2 if seed % 2 == 0 else qrdm
    r = fn(A)
    from oracle import qrdm_oracle as O
    ref = (O.qrdm2 if seed % 2 == 0 else O.qrdm)(A)
    d = np.flatnonzero(r.perm.forward != ref.forward)
    print("seed", seed, (m, n), "rank", r.rank, ref.rank, "first diff", d[:5], "finite", np.isfinite(r.packed).all(),
          [(s.n_s, s.k_selected, s.k_accepted, s.fell_back_to_scalar) for s in r.step_log][:6],
          [(s.n_s, s.k_selected, s.k_accepted, s.fell_back_to_scalar) for s in ref.steps][:6], flush=True)
