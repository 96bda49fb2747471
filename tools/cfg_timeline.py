"""Per-kernel device spans of the last 64 DM steps (DMQR_TIMELINE): mean us per
kernel and the step wall span.  python tools/cfg_timeline.py cfg5 [n] [max_steps]"""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["DMQR_TIMELINE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_03138_b200 import _lib, inputs, rrqr  # noqa: E402

NAMES = {0: "select", 1: "gram", 2: "gram_finish", 3: "swap", 4: "panel_cq", 5: "spare", 6: "ygemm",
         7: "trail_w", 8: "trail_a", 9: "guard", 10: "step_end", 11: "trail_b", 12: "downdate", 13: "panel_rr"}
name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else None
ms = int(sys.argv[3]) if len(sys.argv) > 3 else 0
A = inputs.device_cfg(name, seed=4 if name != "cfg2" else 1, n=n)
work = rrqr.to_work(A)
buf0 = work[0].clone()
for _ in range(2):
    work[0].copy_(buf0)
    f = rrqr.factorize(None, work=work, max_steps=ms)
    torch.cuda.synchronize()
tl_all = np.zeros(64 * 32 + 1024, dtype=np.int64)
_lib.load().dmqr_debug_timeline(f.workspace.data_ptr(), int(A.shape[0]), int(A.shape[1]), tl_all.ctypes.data_as(C.c_void_p))
tl = tl_all[:2048].reshape(64, 16, 2).astype(np.float64)
sp = tl_all[2048:].reshape(256, 4).astype(np.float64)
ok = (tl[:, :, 0] > 0) & (tl[:, :, 0] < 2 ** 62) & (tl[:, :, 1] > 0)
dur = np.where(ok, tl[:, :, 1] - tl[:, :, 0], np.nan) / 1e3
st = np.where(ok, tl[:, :, 0], np.nan)
en = np.where(ok, tl[:, :, 1], np.nan)
span = (np.nanmax(en, axis=1) - np.nanmin(st, axis=1)) / 1e3
print(f"{name}: steps {int(f.info.n_steps)}; last 64 step slots: mean step span {np.nanmean(span):.1f} us")
for k in range(14):
    if np.any(ok[:, k]):
        print(f"  {str(NAMES.get(k, k)):12s} mean {np.nanmean(dur[:, k]):8.1f} us  (in {int(ok[:, k].sum())} steps)")

# k_spare phases (slots 14/15): Q1 seen (first CTA), phase 1 end (last tile), phase 2 end (last CTA out)
sp0 = st[:, 5]
q1 = np.where(ok[:, 14], tl[:, 14, 0], np.nan)
p1 = np.where(tl[:, 14, 1] > 0, tl[:, 14, 1], np.nan)
p2 = np.where(tl[:, 15, 1] > 0, tl[:, 15, 1], np.nan)
pe = en[:, 4]
print("  k_spare (us from its start): phase-1 end %.1f, Q1 seen %.1f, phase-2 end %.1f; panel end %.1f" % (
    np.nanmean(p1 - sp0) / 1e3, np.nanmean(q1 - sp0) / 1e3, np.nanmean(p2 - sp0) / 1e3, np.nanmean(pe - sp0) / 1e3))

# step 20: per-CTA phase-2 view of k_spare (Q1 seen, first G item start, loop exit, items)
v = sp[sp[:, 0] > 0]
if len(v):
    t0 = np.nanmin(v[:, 0])
    print("  step 20 k_spare phase 2 over %d CTAs (us from the first Q1 seen): Q1 seen max %.1f, first item start "
          "mean %.1f, loop exit mean %.1f max %.1f, items mean %.2f max %d" % (
              len(v), (v[:, 0].max() - t0) / 1e3, (v[v[:, 1] > 0, 1].mean() - t0) / 1e3, (v[:, 2].mean() - t0) / 1e3,
              (v[:, 2].max() - t0) / 1e3, v[:, 3].mean(), int(v[:, 3].max())))
