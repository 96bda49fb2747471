"""Device timing of qrp (blocked scalar-pivot engine) on an n x n N(0,1) matrix.

  python tools/qrp_timing.py [n ...]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03138_b200 import _lib, rrqr  # noqa: E402


def main():
    for n in [int(x) for x in sys.argv[1:]] or [4096]:
        g = torch.Generator(device="cuda")
        g.manual_seed(1)
        A = torch.randn(n, n, generator=g, dtype=torch.float64, device="cuda").T
        work = rrqr.to_work(A)
        buf0 = work[0].clone()
        best = 1e30
        for rep in range(3):
            work[0].copy_(buf0)
            torch.cuda.synchronize()
            _lib.load().dmqr_stats_enable(1)
            _lib.stats(reset=True)
            t0 = time.perf_counter()
            f = rrqr.factorize(None, work=work, algo="qrp")
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
            st = _lib.stats(reset=True)
            _lib.load().dmqr_stats_enable(0)
        fl = 2.0 * n ** 3 - 2.0 * n ** 3 / 3.0
        # one read of the trailing block per column: sum_s 8 (n-s)^2 bytes
        rd = sum(8.0 * (n - s) ** 2 for s in range(n))
        print(f"qrp {n}x{n}: {best * 1e3:.1f} ms ({1e6 * best / n:.1f} us/column), {fl / best / 1e9:.0f} GFLOP/s, "
              f"trailing-read floor {rd / 6542.4e9 * 1e3:.1f} ms at 6542 GB/s, rank {int(f.info.rank)}, "
              f"ms_pivot {st['ms_pivot']:.1f}")


if __name__ == "__main__":
    main()
