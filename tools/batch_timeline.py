"""Per-kernel spans of the batched small-matrix path (DMQR_TIMELINE): one lane,
one group of 128 cfg3 matrices.  python tools/batch_timeline.py"""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["DMQR_TIMELINE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_03138_b200 import _lib, inputs  # noqa: E402
from paper_2106_03138_b200.batch import factorize_batch, to_batch_work  # noqa: E402

NAMES = {0: "select", 1: "gram", 2: "gram_finish", 3: "swap", 4: "panel_cq", 5: "spare", 6: "ygemm",
         7: "trail_w", 8: "trail_a", 9: "guard", 10: "step_end", 11: "trail_b", 12: "downdate", 13: "panel_rr"}
w = to_batch_work(inputs.cfg3(seed=3, batch=128), torch.device("cuda"))
for _ in range(2):
    f = factorize_batch(None, lanes=1, work=(w[0].clone(), w[1], w[2], w[3]))
    torch.cuda.synchronize()
tl = np.zeros(64 * 32 + 1024, dtype=np.int64)
_lib.load().dmqr_debug_timeline(tl.ctypes.data_as(C.c_void_p))
tl = tl[:2048].reshape(64, 16, 2).astype(np.float64)
ok = (tl[:, :, 0] > 0) & (tl[:, :, 0] < 2 ** 62) & (tl[:, :, 1] > 0)
for s in range(10):
    if not ok[s].any():
        continue
    t0 = np.min(np.where(ok[s], tl[s, :, 0], np.inf))
    parts = [f"{NAMES[k]}[{(tl[s, k, 0] - t0) / 1e3:.0f},{(tl[s, k, 1] - t0) / 1e3:.0f}]" for k in range(14) if ok[s, k]]
    print(s, " ".join(parts))
