"""Per-reflector phase clocks of one panel CTA (debug; GPU box)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

from paper_2106_03138_b200 import _lib, inputs, rrqr

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cta = int(sys.argv[2]) if len(sys.argv) > 2 else 1
A = inputs.cfg2(seed=1, n=n)
lib = _lib.load()
lib.dmqr_stats_enable(2 + cta)
f = rrqr.factorize(A, max_steps=3)
lib.dmqr_stats_enable(0)
out = np.zeros(64 * 16, dtype=np.int64)
lib.dmqr_debug_panel_clocks(f.workspace.data_ptr(), n, n, out.ctypes.data_as(C.c_void_p))
t = out.reshape(64, 16).astype(np.float64)
order = [0, 5, 6, 7, 1, 8, 9, 10, 11, 2, 3, 4]
names = {0: "start", 5: "vbuf+sync", 6: "vr+dots", 7: "shfl+store", 1: "abc", 8: "sync", 9: "push",
         10: "cluster.sync", 11: "sum", 2: "sync", 3: "update+beta", 4: "T"}
rows = t[2:60]
prev = order[0]
res = {}
for ph in order[1:]:
    res[names[ph]] = float(np.median(rows[:, ph] - rows[:, prev]))
    prev = ph
print("cta", cta, "median cycles:", res)
print("round (start->T):", float(np.median(rows[:, 4] - rows[:, 0])),
      " start->next start:", float(np.median(rows[1:, 0] - rows[:-1, 0])))
