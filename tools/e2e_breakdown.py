"""Where the end-to-end qrdm2 call spends its time (host-timed pieces).

  python tools/e2e_breakdown.py [--size 4096]
"""

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_03138_b200 import inputs, rrqr  # noqa: E402


def tick(label, t0, out):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out.append((label, (t - t0) * 1e3))
    return t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    A = inputs.cfg2(seed=1, n=a.size)
    pinned = torch.from_numpy(np.ascontiguousarray(A)).pin_memory()
    for rep in range(a.reps):
        out = []
        torch.cuda.synchronize()
        t = t0 = time.perf_counter()
        work = rrqr.to_work(pinned)
        t = tick("to_work (H2D + transpose)", t, out)
        f = rrqr.factorize(None, work=work)
        t = tick("factorize", t, out)
        steps = rrqr._steps_from_raw(f.steps.cpu().numpy(), int(f.info.n_steps))
        t = tick("steps D2H + parse", t, out)
        sw = f.swaps[: int(f.info.n_swaps)].cpu().numpy()
        t = tick("swaps D2H", t, out)
        _ = [(int(x), int(y)) for x, y in sw]
        t = tick("swaps to list", t, out)
        host = f.buf[: f.n, : f.m]
        h = host.cpu() if host.is_contiguous() else host.contiguous().cpu()
        t = tick(f"packed D2H pageable (contig={host.is_contiguous()})", t, out)
        pin = torch.empty(host.shape, dtype=host.dtype, pin_memory=True)
        t = tick("alloc pinned", t, out)
        pin.copy_(host)
        t = tick("packed D2H pinned", t, out)
        _ = rrqr.replay_counters(f.m, f.n, steps)
        t = tick("replay_counters", t, out)
        r = rrqr.qrdm2(pinned)
        t = tick("qrdm2 total", t, out)
        print(f"rep {rep}: " + ", ".join(f"{k} {v:.2f}" for k, v in out), flush=True)
        del h, pin, r


if __name__ == "__main__":
    main()
