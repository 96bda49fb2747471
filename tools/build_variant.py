"""Build an A/B variant of the library with extra -D flags into _ab/<name>.so:
python tools/build_variant.py r32n2 -DDMQR_TA_ROWS=32 -DDMQR_TA_NST=2
(load it with DMQR_LIB_PATH=_ab/<name>.so)"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2106_03138_b200 import _build  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = ROOT / "_ab" / f"{name}.so"
out.parent.mkdir(exist_ok=True)
subprocess.run([_build.NVCC, *_build.FLAGS, *defs, "-o", str(out), str(_build.CSRC / "dmqr_b200.cu")], check=True)
print(out)
