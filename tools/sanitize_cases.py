"""Small factorizations covering every kernel family, for compute-sanitizer:
  compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_cases.py [quick]
fused small kernel, per-step kernels, look-ahead schedule (k_spare / k_trail_w /
k_guard), tall panel helpers, Householder panel, blocked scalar pivoting
(k_qp3, qrp and a QRDM fallback run), batched groups, explicit Q."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2106_03138_b200 import qrdm, qrdm2, qrp, reconstruct  # noqa: E402
from paper_2106_03138_b200.batch import factorize_batch  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
rng = np.random.default_rng(3)


def run(label, fn, A, env=None):
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        r = fn(A)
        Q, R = reconstruct(r)
        res = np.linalg.norm(A[:, r.perm.forward] - Q @ R) / np.linalg.norm(A)
        print(f"{label}: rank {r.rank} steps {len(r.step_log)} resid {res:.1e}", flush=True)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


graded = lambda m, n: rng.standard_normal((m, n)) * np.logspace(0, -10, n)[rng.permutation(n)]  # noqa: E731
run("fused small 200x150", qrdm2, graded(200, 150))
run("step kernels 200x150", qrdm2, graded(200, 150), {"DMQR_NO_FUSED": "1"})
run("qrdm 300x260", qrdm, graded(300, 260))
run("lookahead 1100x1024", qrdm2, graded(1100, 1024))
if not quick:
    run("householder panel 1100x1024", qrdm2, graded(1100, 1024), {"DMQR_NO_CHOLQR": "1"})
    run("tall helpers 9000x256", qrdm2, graded(9000, 256))
    A = rng.standard_normal((600, 500)) @ np.diag(np.logspace(0, -30, 500)) @ rng.standard_normal((500, 500))
    run("fallback run 600x500", qrdm2, A)
    run("qrp 700x600", qrp, graded(700, 600))
B = rng.standard_normal((5, 128, 96))
f = factorize_batch(B)
print("batched fused ranks", [f.result(i).rank for i in range(5)])
os.environ["DMQR_NO_FUSED"] = "1"
f = factorize_batch(B)
print("batched groups ranks", [f.result(i).rank for i in range(5)], flush=True)
