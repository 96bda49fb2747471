"""Phase clocks of one k_qp3 block (CTA 0, globaltimer ns).

  python tools/qp_clocks.py [n] [block]      # qrp on n x n N(0,1), block index (default 2)
"""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_03138_b200 import _lib, rrqr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g = torch.Generator(device="cuda")
g.manual_seed(1)
A = torch.randn(n, n, generator=g, dtype=torch.float64, device="cuda").T
work = rrqr.to_work(A)
buf0 = work[0].clone()
rrqr.factorize(None, work=work, algo="qrp")  # warm
work[0].copy_(buf0)
os.environ["DMQR_QP_CLOCKS"] = str(blk)
f = rrqr.factorize(None, work=work, algo="qrp")
torch.cuda.synchronize()
out = np.zeros(64 * 16, dtype=np.int64)
_lib.load().dmqr_debug_panel_clocks(f.workspace.data_ptr(), n, n, out.ctypes.data_as(C.c_void_p))
ph = out[:512].reshape(64, 8).astype(np.float64)
names = ["guard wait", "gamma (argmax, swap, pivot col) + B1", "alpha reduce+w loop+B2 ... ", "beta + B3", "guard"]
d = np.diff(np.concatenate([ph[:, :5], ph[1:, :1].tolist() + [[np.nan]]], axis=1), axis=1)
print(f"qrp {n}x{n}, block {blk} (columns {64 * blk}..): mean us per column")
labels = ["0->1 guard-done wait", "1->2 gamma+B1", "2->3 alpha+B2", "3->4 beta+B3", "4->next guard phase"]
for i, l in enumerate(labels):
    col = d[:63, i] / 1e3
    print(f"  {l:24s} {np.nanmean(col):8.2f}  (min {np.nanmin(col):.2f}, max {np.nanmax(col):.2f})")
tot = (ph[63, 0] - ph[0, 0]) / 63 / 1e3
print(f"  per column total         {tot:8.2f}")
print(f"  block end: Wt build {(out[513] - out[512]) / 1e3:.1f} us, tiles {(out[514] - out[513]) / 1e3:.1f} us")
