"""Debug aid: one cfg1 qrdm factorization vs the golden permutation (PKGROOT selects a build)."""
import os
import sys
sys.path[:0] = [os.environ.get("PKGROOT", "/root/repo"), "/root/repo", "/root/repo/tests"]
import numpy as np  # noqa: E402

import golden_cases as G  # noqa: E402
from paper_2106_03138_b200 import qrdm  # noqa: E402

A = G.case_input("cfg1/qrdm")
r = qrdm(A)
d = np.flatnonzero(r.perm.forward != G.case_field("cfg1/qrdm", "forward"))
print("rank", r.rank, "first diff", d[:5], [(s.n_s, s.k_selected, s.k_accepted) for s in r.step_log][:4], flush=True)
