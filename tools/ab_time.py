"""A/B device timing of one cfg2-style factorization (CUDA events, stats off),
run from a repo checkout: python tools/ab_time.py [n] [reps] [cfg]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path.cwd()))
import torch  # noqa: E402

from paper_2106_03138_b200 import inputs, rrqr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = sys.argv[3] if len(sys.argv) > 3 else "cfg2"
A = inputs.device_cfg(cfg, seed=1 if cfg == "cfg2" else 4, n=n)
work = rrqr.to_work(A)
buf0 = work[0].clone()
ts = []
for r in range(reps + 1):
    work[0].copy_(buf0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f = rrqr.factorize(None, work=work)
    e1.record()
    torch.cuda.synchronize()
    if r:
        ts.append(e0.elapsed_time(e1))
if ts:
    print(f"{Path.cwd().name} {cfg} n={n}: best {min(ts):.2f} ms median {sorted(ts)[len(ts) // 2]:.2f} ms rank {int(f.info.rank)}")
