"""Chunked CholeskyQR2 panel vs the Householder panel after one step (debug)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_03138_b200 import rrqr  # noqa: E402

m = int(sys.argv[1]); n = int(sys.argv[2]); steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
gen = torch.Generator(device="cuda")
gen.manual_seed(7)
A = torch.randn(m, n, generator=gen, dtype=torch.float64, device="cuda")
os.environ["DMQR_NO_LOOKAHEAD"] = "1"
a = rrqr.to_result(rrqr.factorize(A.clone(), max_steps=steps))
os.environ["DMQR_NO_CHOLQR"] = "1"
b = rrqr.to_result(rrqr.factorize(A.clone(), max_steps=steps))
d = np.abs(a.packed - b.packed)
print(m, n, "steps", [(s.n_s, s.k_selected, s.k_accepted) for s in a.step_log],
      [(s.n_s, s.k_selected, s.k_accepted) for s in b.step_log])
print("max |diff|", d.max(), "coeffs diff", np.abs(a.coeffs - b.coeffs).max())
if d.max() > 1e-8:
    i, j = np.unravel_index(d.argmax(), d.shape)
    print("worst", i, j, a.packed[i, j], b.packed[i, j])
    rows = np.where(d.max(axis=1) > 1e-8)[0]
    print("bad rows", rows[:10], rows[-10:], len(rows))
cn = torch.linalg.norm(A, dim=0)
p = int(torch.argmax(cn))
print("max col norm", float(cn[p]), "col", p, "x0 sign", float(torch.sign(A[0, p])), "cq R00", a.packed[0, 0], "hh R00", b.packed[0, 0],
      "perm0", a.perm.forward[0], b.perm.forward[0])
