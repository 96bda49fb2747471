"""Finer host-timed split of the public qrdm2(pinned host tensor) call (the bench's e2e path):
to_work's pieces, the pinned result buffer, factorize (engine + streamed D2H), to_result.

  python tools/e2e_fine.py [--size 4096]
"""

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_03138_b200 import inputs, rrqr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    A = inputs.cfg2(seed=1, n=a.size)
    pinned = torch.from_numpy(np.ascontiguousarray(A)).pin_memory()
    dev = torch.device("cuda", 0)

    def now():
        torch.cuda.synchronize()
        return time.perf_counter()

    for rep in range(a.reps):
        out = []
        t0 = t = now()
        td = pinned.to(device=dev, dtype=torch.float64)
        t1 = now(); out.append(("H2D", t1 - t)); t = t1
        m, n = td.shape
        lda = rrqr.lda_for(m)
        buf = torch.zeros((n, lda), dtype=torch.float64, device=dev)
        t1 = now(); out.append(("zeros", t1 - t)); t = t1
        buf[:n, :m].copy_(td.T)
        t1 = now(); out.append(("transpose", t1 - t)); t = t1
        hp = torch.empty((n, m), dtype=torch.float64, pin_memory=True)
        t1 = now(); out.append(("pinned alloc", t1 - t)); t = t1
        f = rrqr.factorize(None, work=(buf, m, n, lda), host_packed=hp, algo="qrdm")
        t1 = now(); out.append(("factorize+stream", t1 - t)); t = t1
        r = rrqr.to_result(f)
        t1 = now(); out.append(("to_result", t1 - t)); t = t1
        out.append(("sum", t - t0))
        t = now()
        r2 = rrqr.qrdm2(pinned)
        out.append(("qrdm2 total", now() - t))
        print(f"rep {rep}: " + ", ".join(f"{k} {v * 1e3:.3f}" for k, v in out), flush=True)
        del r, r2, f, hp, buf, td


if __name__ == "__main__":
    main()
