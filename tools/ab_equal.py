"""A/B of two library builds in separate processes: time + sha256 of the packed factor.
  python tools/ab_equal.py <n|cfg:n> [env=val ...]   (DMQR_LIB_PATH selects the build)"""
import hashlib
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path.cwd()))
for kv in sys.argv[2:]:
    k, v = kv.split("=", 1)
    os.environ[k] = v
import torch  # noqa: E402

from paper_2106_03138_b200 import inputs, rrqr  # noqa: E402

arg = sys.argv[1]
cfg, n = arg.split(":") if ":" in arg else ("cfg2", arg)
n = int(n)
A = inputs.device_cfg(cfg, seed=1 if cfg == "cfg2" else 4, n=n)
work = rrqr.to_work(A)
buf0 = work[0].clone()
ts = []
for r in range(4):
    work[0].copy_(buf0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f = rrqr.factorize(None, work=work)
    e1.record()
    torch.cuda.synchronize()
    if r:
        ts.append(e0.elapsed_time(e1))
h = hashlib.sha256(work[0].cpu().numpy().tobytes()).hexdigest()[:16]
print(f"{os.environ.get('DMQR_LIB_PATH', 'HEAD'):14s} {arg:12s} {' '.join(sys.argv[2:]):24s} best {min(ts):8.2f} ms  rank {int(f.info.rank)} "
      f"steps {int(f.info.n_steps)} sha {h}", flush=True)
