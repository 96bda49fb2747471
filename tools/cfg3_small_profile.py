"""cfg3 batch through the fused small-matrix kernel once (ncu target): python tools/cfg3_small_profile.py [batch]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03138_b200 import inputs  # noqa: E402
from paper_2106_03138_b200.batch import factorize_batch, to_batch_work  # noqa: E402

batch = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
w = to_batch_work(inputs.cfg3(seed=3, batch=batch))
f = factorize_batch(None, work=w)
torch.cuda.synchronize()
print("ranks", sorted(set(f.ranks.tolist())))
