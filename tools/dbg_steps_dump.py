"""Debug aid: packed factor of cfg1 after 1 and 2 outer steps (PKGROOT selects a build) -> npz."""
import os
import sys
sys.path[:0] = [os.environ.get("PKGROOT", "/root/repo"), "/root/repo", "/root/repo/tests"]
import numpy as np  # noqa: E402

import golden_cases as G  # noqa: E402
from paper_2106_03138_b200 import rrqr  # noqa: E402

A = G.case_input("cfg1/qrdm")
out = {}
for ms in (1, 2):
    f = rrqr.factorize(A, break_check=False, max_steps=ms)
    r = rrqr.to_result(f)
    out[f"packed{ms}"] = np.asarray(r.packed)
    out[f"perm{ms}"] = np.asarray(r.perm.forward)
    out[f"coeffs{ms}"] = np.asarray(r.coeffs)
    out[f"T{ms}"] = f.workspace[:].cpu().numpy()[:0]
np.savez(sys.argv[1], **out)
print("saved", sys.argv[1])
