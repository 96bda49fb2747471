"""Phase cycles of the fused small-matrix kernel (CTA 0) on the cfg3 batch:
DMQR_SMALL_CLOCKS=1 python tools/small_clocks.py"""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ["DMQR_SMALL_CLOCKS"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_03138_b200 import _lib, inputs  # noqa: E402
from paper_2106_03138_b200.batch import factorize_batch, to_batch_work  # noqa: E402

NAMES = ["init norms", "argmax/stop", "candidates", "gather", "cosine gram", "filter+gamma", "swap plan", "moves",
         "compaction", "panel", "writeback", "Y fix + S", "T", "trailing", "downdate+record", "fallback steps"]
w = to_batch_work(inputs.cfg3(seed=3, batch=1024))
f = factorize_batch(None, work=w)
torch.cuda.synchronize()
out = np.zeros(32, dtype=np.int64)
_lib.load().dmqr_debug_small_clocks(out.ctypes.data_as(C.c_void_p))
tot = out.sum()
per = -(-1024 // 148)
print(f"CTA 0: {tot} cycles over ~{per} matrices ({tot / 1.965e3:.0f} us)")
print('panel j=16 owner of 17 (step 0): wait / vq / apply / ring / reflector / publish / batch end:', out[16:23].tolist())
print('moves split (thread-0 lists / u,perm / data):', (out[23:26] / per / 1.965e3).round(1).tolist(), 'us/matrix')
for nm, v in zip(NAMES, out[:16]):
    print(f"  {nm:16s} {v:12d}  {100 * v / max(tot, 1):5.1f}%  {v / per / 1.965e3:8.1f} us/matrix")
