"""A few outer steps of cfg2 (for ncu captures of the panel kernels)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2106_03138_b200 import inputs, rrqr
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
A = inputs.cfg2(seed=1, n=n)
f = rrqr.factorize(A, max_steps=steps)
torch.cuda.synchronize()
print("ok", f.info.n_steps)
