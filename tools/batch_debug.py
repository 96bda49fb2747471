import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2106_03138_b200 import inputs
from paper_2106_03138_b200.batch import factorize_batch
B = inputs.cfg3(seed=3, batch=int(sys.argv[1]) if len(sys.argv) > 1 else 2)
try:
    f = factorize_batch(B, lanes=1)
    print("ok", [int(i.rank) for i in f.infos])
except Exception as e:
    print("ERR", e)
