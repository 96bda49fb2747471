"""Loader for the committed golden vectors (tests/golden/golden.npz + index)."""

from __future__ import annotations

import hashlib
import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=1)
def index() -> dict:
    return json.loads((GOLDEN / "golden_index.json").read_text())


@lru_cache(maxsize=1)
def store():
    return np.load(GOLDEN / "golden.npz")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.float64)).tobytes(order="C")).hexdigest()


@lru_cache(maxsize=1)
def _fixtures() -> dict:
    import fixture_suite
    return dict(fixture_suite.suite())


@lru_cache(maxsize=8)
def _cfg3_small():
    from paper_2106_03138_b200 import inputs
    return inputs.cfg3(seed=3, batch=4)


def case_input(name: str) -> np.ndarray:
    """Regenerate (or load) the input of a golden case."""
    meta = index()["cases"][name]
    if meta.get("input"):
        return np.array(store()[f"{name}/input"])
    from paper_2106_03138_b200 import inputs
    src = meta["source"]
    if src.startswith("wide:"):
        import wide_cases
        return wide_cases.make(src[5:])
    if src == "fixture":
        parts = name.split("/")
        return _fixtures()[parts[2] if parts[0] == "qrp" else parts[1]]
    if src.startswith("inputs.cfg1"):
        return inputs.cfg1(seed=0)
    if src.startswith("inputs.cfg2"):
        return inputs.cfg2(seed=1, n=1024)
    if src.startswith("inputs.cfg3"):
        return _cfg3_small()[int(src.split("[")[1].rstrip("]"))]
    if src.startswith("inputs.cfg4"):
        return inputs.cfg4(seed=4, m=8192, n=256)
    if src.startswith("inputs.cfg5"):
        return inputs.cfg5(seed=4, n=1024)
    raise KeyError(src)


def case_field(name: str, field: str):
    return store()[f"{name}/{field}"]


def case_names(prefix: str = "") -> list:
    return sorted(k for k in index()["cases"] if k.startswith(prefix))


def oracle_kwargs(name: str) -> dict:
    meta = index()["cases"][name]
    return dict(tau=meta["tau"], delta=meta["delta"], k_dm=meta["k_dm"],
                use_delta_max=meta["use_delta_max"], stop_rule=meta["stop"])
