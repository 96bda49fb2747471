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

cfg5 = len(sys.argv) > 1 and sys.argv[1] == "cfg5"   # qrdm2 on cfg5: the blocks of its fallback run
n = 16384 if cfg5 else (int(sys.argv[1]) if len(sys.argv) > 1 else 4096)
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if cfg5:
    from paper_2106_03138_b200 import inputs
    A = inputs.device_cfg("cfg5", seed=4)
else:
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    A = torch.randn(n, n, generator=g, dtype=torch.float64, device="cuda").T
algo = "qrdm" if cfg5 else "qrp"
work = rrqr.to_work(A)
buf0 = work[0].clone()
rrqr.factorize(None, work=work, algo=algo)  # warm
work[0].copy_(buf0)
os.environ["DMQR_QP_CLOCKS"] = str(blk)
f = rrqr.factorize(None, work=work, algo=algo)
torch.cuda.synchronize()
out = np.zeros(64 * 16, dtype=np.int64)
_lib.load().dmqr_debug_panel_clocks(f.workspace.data_ptr(), n, n, out.ctypes.data_as(C.c_void_p))
ph = out[:512].reshape(64, 8).astype(np.float64)
# valid columns: increasing stamps from the first one (the workspace is not zeroed)
nv = 0
while nv < 64 and ph[nv, 0] > 0 and (nv == 0 or 0 < ph[nv, 0] - ph[nv - 1, 0] < 1e8):
    nv += 1
print(f"{'cfg5 qrdm fallback run' if cfg5 else f'qrp {n}x{n}'}, block {blk}: {nv} columns; mean us per column")
if nv >= 2:
    d = np.diff(np.concatenate([ph[:nv - 1, :5], ph[1:nv, :1]], axis=1), axis=1) / 1e3
    labels = ["0->1 guard-done wait", "1->2 gamma+B1", "2->3 alpha+B2", "3->4 beta+B3", "4->next guard phase"]
    for i, l in enumerate(labels):
        print(f"  {l:24s} {np.mean(d[:, i]):8.2f}  (min {np.min(d[:, i]):.2f}, max {np.max(d[:, i]):.2f})")
    print(f"  per column total         {(ph[nv - 1, 0] - ph[0, 0]) / (nv - 1) / 1e3:8.2f}")
print(f"  block end: Wt build {(out[513] - out[512]) / 1e3:.1f} us, tiles {(out[514] - out[513]) / 1e3:.1f} us")
