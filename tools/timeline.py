"""Per-step panel vs k_spare timing from globaltimer stamps (DMQR_TIMELINE=1)."""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["DMQR_TIMELINE"] = "1"
import numpy as np  # noqa: E402

from paper_2106_03138_b200 import _lib, inputs, rrqr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
A = inputs.cfg2(seed=1, n=n)
work = rrqr.to_work(A)
buf0 = work[0].clone()
for _ in range(2):
    work[0].copy_(buf0)
    f = rrqr.factorize(None, work=work)
out = np.zeros(64 * 16, dtype=np.int64)
_lib.load().dmqr_debug_panel_clocks(f.workspace.data_ptr(), n, n, out.ctypes.data_as(C.c_void_p))
t = out.reshape(-1, 4)[: int(f.info.n_steps)]
print("step  panel_us  spare_start_us  spare_end_us  (relative to the panel start)")
for i, (p0, p1, s0, s1) in enumerate(t):
    if p0 == 0:
        continue
    print(f"{i:4d} {(p1 - p0) / 1e3:9.1f} {(s0 - p0) / 1e3:14.1f} {(s1 - p0) / 1e3:13.1f}")
g = out[512:512 + 8 * 64].reshape(64, 8)[: int(f.info.n_steps)]
print("gram_finish (us from CTA entry): last-CTA start, loaded, Theta start, filter start, plan start, end, masks done, greedy done")
for i, r in enumerate(g[:12]):
    if r[0] == 0:
        continue
    print(i, [round(float(x - r[0]) / 1e3, 1) if x else None for x in r[1:8]])
