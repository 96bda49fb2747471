import ctypes as C, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2106_03138_b200 import _lib, inputs, rrqr
A = inputs.device_cfg("cfg4", seed=4)
lib = _lib.load()
for cta in (0, 1):
    lib.dmqr_stats_enable(2 + cta)
    f = rrqr.factorize(A, max_steps=3)
    torch.cuda.synchronize()
    lib.dmqr_stats_enable(0)
    out = np.zeros(64 * 16, dtype=np.int64)
    lib.dmqr_debug_panel_clocks(f.workspace.data_ptr(), 65536, 1024, out.ctypes.data_as(C.c_void_p))
    t = out[:24].astype(np.float64)
    names = ["load", "gram1", "reduce1", "chol1", "trinv1", "Q1gemm", "gram2", "reduce2", "R2", "break", "trinvR2",
             "Qtop", "mLU", "UY+sync", "T", "aux", "end"]
    d = np.diff(t)
    print("cta", cta, {names[i]: int(v) for i, v in enumerate(d[:17]) if abs(v) < 1e9}, "total", int(t[17] - t[0]) if 0 < t[17] - t[0] < 1e10 else None)
