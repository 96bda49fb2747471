"""cfg5 time split: DM steps vs the scalar-fallback run (device inputs).

  python tools/cfg5_split.py [n]

Factors cfg5 fully, reads the step log, then re-runs with max_steps = index of
the first fallback step; the difference is the fallback run's time.
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03138_b200 import _lib, inputs, rrqr  # noqa: E402


def run(work, buf0, max_steps=0, reps=2):
    best = 1e30
    f = None
    for _ in range(reps):
        work[0].copy_(buf0)
        torch.cuda.synchronize()
        _lib.load().dmqr_stats_enable(1)
        _lib.stats(reset=True)
        t0 = time.perf_counter()
        f = rrqr.factorize(None, work=work, max_steps=max_steps)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
        st = _lib.stats(reset=True)
        _lib.load().dmqr_stats_enable(0)
    return best, f, st


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else None
    A = inputs.device_cfg("cfg5", seed=4, n=n)
    work = rrqr.to_work(A)
    buf0 = work[0].clone()
    t, f, st = run(work, buf0)
    steps = rrqr._steps_from_raw(f.steps.cpu().numpy(), int(f.info.n_steps))
    fb = [i for i, s in enumerate(steps) if s.fell_back_to_scalar]
    print(f"full: {t * 1e3:.1f} ms, steps {len(steps)}, fallback steps {len(fb)}, rank {int(f.info.rank)}, "
          + ", ".join(f"{k} {st[k]:.1f}" for k in ("ms_select", "ms_panel", "ms_trailing", "ms_norms")))
    if fb:
        i0 = fb[0]
        print(f"first fallback step {i0} (n_s {steps[i0].n_s}), last {fb[-1]} (n_s {steps[fb[-1]].n_s}); "
              f"DM steps after the run: {len(steps) - 1 - fb[-1]}")
        t1, _, st1 = run(work, buf0, max_steps=i0)
        print(f"up to the fallback run: {t1 * 1e3:.1f} ms, "
              + ", ".join(f"{k} {st1[k]:.1f}" for k in ("ms_select", "ms_panel", "ms_trailing", "ms_norms")))
        t2, _, st2 = run(work, buf0, max_steps=fb[-1] + 1)
        print(f"through the fallback run: {t2 * 1e3:.1f} ms -> fallback run {1e3 * (t2 - t1):.1f} ms "
              f"({1e6 * (t2 - t1) / len(fb):.0f} us/step); "
              + ", ".join(f"{k} {st2[k] - st1[k]:.1f}" for k in ("ms_select", "ms_panel", "ms_trailing",
                                                                  "ms_norms")))


if __name__ == "__main__":
    main()
