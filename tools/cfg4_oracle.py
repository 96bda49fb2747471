"""cfg4-like tall matrix: GPU step log (look-ahead, serial) vs the CPU oracle (debug)."""
import os
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
nsteps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
import torch  # noqa: E402

gen = torch.Generator(device="cuda")
gen.manual_seed(4)
q, r = torch.linalg.qr(torch.randn(m, n, generator=gen, dtype=torch.float64, device="cuda"))
U = q * torch.sign(torch.diagonal(r))
V, _ = torch.linalg.qr(torch.randn(n, n, generator=gen, dtype=torch.float64, device="cuda"))
s = torch.arange(1, n + 1, dtype=torch.float64, device="cuda") ** -2.0
A = (U * s) @ V.T
A *= 10.0 ** (torch.rand(n, generator=gen, dtype=torch.float64, device="cuda") * 6.0 - 6.0)
Ah = np.asfortranarray(A.cpu().numpy())

from paper_2106_03138_b200 import rrqr  # noqa: E402
from oracle import qrdm_oracle as O  # noqa: E402


def log_of(steps):
    return [(st.n_s, st.k_selected, st.k_accepted, int(st.broke_early)) for st in steps]


la = rrqr.to_result(rrqr.factorize(A.clone()))
os.environ["DMQR_NO_LOOKAHEAD"] = "1"
se = rrqr.to_result(rrqr.factorize(A.clone()))
os.environ["DMQR_NO_CHOLQR"] = "1"
hh = rrqr.to_result(rrqr.factorize(A.clone()))
del os.environ["DMQR_NO_CHOLQR"]
del os.environ["DMQR_NO_LOOKAHEAD"]
t0 = time.time()
ref = O.qrdm2(Ah, max_steps=nsteps, margins=True)
print("oracle", time.time() - t0, "s")
print("oracle", log_of(ref.steps)[:nsteps])
print("la    ", log_of(la.step_log)[:nsteps])
print("serial", log_of(se.step_log)[:nsteps])
print("hh    ", log_of(hh.step_log)[:nsteps])
print("margins", ref.margins["per_step"][:nsteps] if isinstance(ref.margins, dict) else ref.margins)
