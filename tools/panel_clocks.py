"""Per-reflector phase clocks of one panel CTA (debug; GPU box)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_2106_03138_b200 import _lib, inputs, rrqr

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
A = inputs.cfg2(seed=1, n=n)
lib = _lib.load()
lib.dmqr_stats_enable(2)
f = rrqr.factorize(A, max_steps=3)
lib.dmqr_stats_enable(0)
out = np.zeros(64 * 8, dtype=np.int64)
lib.dmqr_debug_panel_clocks(f.workspace.data_ptr(), n, n, out.ctypes.data_as(C.c_void_p))
t = out.reshape(64, 8)[:, :6].astype(np.float64)
d = np.diff(t, axis=1)
names = ["refl+dots+abc", "allreduce", "update", "T", "nextnorm"]
print("median cycles per phase:", {nm: float(np.median(d[1:60, i])) for i, nm in enumerate(names)})
per = np.diff(t[:, 0])
print("median cycles per reflector:", float(np.median(per[1:60])))
