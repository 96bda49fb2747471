"""A few outer steps of cfg4 (65536 x 1024; for ncu captures of the tall panel and its helpers)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2106_03138_b200 import inputs, rrqr
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
A = inputs.device_cfg("cfg4", seed=4)
f = rrqr.factorize(A, max_steps=steps)
torch.cuda.synchronize()
print("ok", f.info.n_steps)
