import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2106_03138_b200 import inputs, rrqr
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
A = inputs.cfg2(seed=1, n=n)
for s in (1, 2, 3, 10):
    f = rrqr.factorize(A, max_steps=s)
    d = f.debug_ctl()
    print("step", s, "n_s", d["n_s"], "k_s", d["k_s"], "l_acc", d["l_acc"], "cq_fail*1e6+tc0", int(np.array([d["gamma"]]).view(np.int64)[0]) if False else d)
