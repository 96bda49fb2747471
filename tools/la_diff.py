"""Look-ahead vs serial schedule on a cfg4-like tall matrix: first differing step (debug)."""
import os
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
if os.environ.get("CHILD"):
    import torch

    from paper_2106_03138_b200 import rrqr
    gen = torch.Generator(device="cuda")
    gen.manual_seed(4)
    q, r = torch.linalg.qr(torch.randn(m, n, generator=gen, dtype=torch.float64, device="cuda"))
    U = q * torch.sign(torch.diagonal(r))
    V, _ = torch.linalg.qr(torch.randn(n, n, generator=gen, dtype=torch.float64, device="cuda"))
    s = torch.arange(1, n + 1, dtype=torch.float64, device="cuda") ** -2.0
    A = (U * s) @ V.T
    A *= 10.0 ** (torch.rand(n, generator=gen, dtype=torch.float64, device="cuda") * 6.0 - 6.0)
    f = rrqr.factorize(A)
    res = rrqr.to_result(f)
    log = np.array([(st.n_s, st.k_selected, st.k_accepted, st.broke_early, st.fell_back_to_scalar, st.k_max)
                    for st in res.step_log])
    np.savez(os.environ["CHILD"], log=log, perm=res.perm.forward, packed=res.packed)
    sys.exit(0)
for mode in ("la", "serial"):
    env = dict(os.environ, CHILD=f"/tmp/ld_{mode}.npz")
    if mode == "serial":
        env["DMQR_NO_LOOKAHEAD"] = "1"
    subprocess.run([sys.executable, __file__, str(m), str(n)], env=env, check=True)
a, b = np.load("/tmp/ld_la.npz"), np.load("/tmp/ld_serial.npz")
la, se = a["log"], b["log"]
print("steps", len(la), len(se))
for i in range(min(len(la), len(se))):
    if not np.array_equal(la[i], se[i]):
        print("first diff at step", i, "la", la[i], "serial", se[i])
        print("prev", la[max(0, i - 2):i + 2].tolist(), se[max(0, i - 2):i + 2].tolist())
        break
else:
    print("step logs equal over the common prefix")
print("perm equal", np.array_equal(a["perm"], b["perm"]), "max |dpacked|", np.abs(a["packed"] - b["packed"]).max())
