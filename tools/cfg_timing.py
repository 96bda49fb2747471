"""Device timing of one factorization for the BASELINE configs (device-generated inputs).

  python tools/cfg_timing.py cfg4 [n]     # cfg2 / cfg4 / cfg5
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03138_b200 import _lib, inputs, rrqr  # noqa: E402


def main():
    name = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else None
    A = inputs.device_cfg(name, seed=4 if name != "cfg2" else 1, n=n)
    m, nn = A.shape
    work = rrqr.to_work(A)
    buf0 = work[0].clone()
    lib = _lib.load()
    best = 1e30
    for rep in range(3):
        work[0].copy_(buf0)
        torch.cuda.synchronize()
        lib.dmqr_stats_enable(1)
        _lib.stats(reset=True)
        t0 = time.perf_counter()
        f = rrqr.factorize(None, work=work)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if dt < best:
            best, st = dt, _lib.stats(reset=True)
        else:
            _lib.stats(reset=True)
        lib.dmqr_stats_enable(0)
    flops = 2.0 * m * nn * nn - 2.0 * nn ** 3 / 3.0 if m >= nn else 2.0 * nn * m * m - 2.0 * m ** 3 / 3.0
    dt = best
    print(f"{name} {m}x{nn}: {dt * 1e3:.1f} ms (best of 3), {flops / dt / 1e9:.0f} GFLOP/s, rank {int(f.info.rank)}, "
          f"steps {int(f.info.n_steps)}, phases " + ", ".join(f"{k} {st[k]:.1f}" for k in
                                                              ("ms_select", "ms_panel", "ms_trailing", "ms_norms", "ms_pivot")))


if __name__ == "__main__":
    main()
