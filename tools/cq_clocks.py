"""Phase clocks of the CholeskyQR2 panel kernel (debug; GPU box)."""
import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2106_03138_b200 import _lib, inputs, rrqr
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
A = inputs.cfg2(seed=1, n=n)
lib = _lib.load()
lib.dmqr_stats_enable(2 + cta)
f = rrqr.factorize(A, max_steps=3)
lib.dmqr_stats_enable(0)
out = np.zeros(64 * 16, dtype=np.int64)
lib.dmqr_debug_panel_clocks(f.workspace.data_ptr(), n, n, out.ctypes.data_as(C.c_void_p))
t = out[:24].astype(np.float64)
names = ["load", "gram1", "reduce1", "chol1", "trinv1", "Q1gemm", "gram2", "reduce2", "R2", "break", "trinvR2",
         "Qtop", "mLU", "UY+sync", "T", "aux", "end"]
d = np.diff(t)
print("cta", cta, {names[i] if i < len(names) else i: int(v) for i, v in enumerate(d[:17])}, "total", int(t[17] - t[0]) if t[17] else None)
f = out[32:48]
print("fine (cycles from Q1gemm end):", [int(x - t[6]) if x else None for x in f])
