import os
import sys
from pathlib import Path

# Pin BLAS threads: the oracle's bit-exact pins were made with 1 OpenBLAS thread
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

ROOT = Path(__file__).resolve().parent.parent
for p in (str(ROOT), str(ROOT / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built libdmqr_b200.so")
    config.addinivalue_line("markers", "slow: long-running (large oracle runs)")
