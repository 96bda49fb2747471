"""Algorithm registry wiring.

The reference's harness dispatches by name through ``ALGORITHMS`` and
``run_algorithm`` (harness.py:40, 188-198); its CLI offers ``sorted(ALGORITHMS)``
as ``--algo`` choices (cli.py:46).  This module provides the same two names
backed by the B200 engine, and ``register`` adds ``<name>_b200`` entries to the
reference's own registry so its harness, sweeps and CLI can select the device
path without any other change (INTEGRATION.md shows the two-line hook).
"""

from __future__ import annotations

from .rrqr import DMParams, RRQRResult, StopCriterion, qrdm, qrdm2, qrp

ALGORITHMS = {"qrp": qrp, "qrdm": qrdm, "qrdm2": qrdm2}  # harness.py:40


def run_algorithm(algo: str, A, params: DMParams, stop: StopCriterion, trace_norms: bool = False) -> RRQRResult:
    """harness.run_algorithm (harness.py:188-198) on the B200 engine; KeyError on unknown names."""
    fn = ALGORITHMS[algo]
    if algo == "qrp":
        return fn(A, stop=stop, trace_norms=trace_norms)
    return fn(A, params=params, stop=stop, trace_norms=trace_norms)


def _qrp_entry(A, params: DMParams | None = None, stop: StopCriterion = StopCriterion(),
               trace_norms: bool = False) -> RRQRResult:
    # the reference's run_algorithm passes params= to every name but "qrp"
    return qrp(A, stop=stop, trace_norms=trace_norms)


B200_ALGORITHMS = {"qrp_b200": _qrp_entry, "qrdm_b200": qrdm, "qrdm2_b200": qrdm2}


def register(registry: dict) -> dict:
    """Add the ``*_b200`` entries to a reference-style ``ALGORITHMS`` dict (in place)."""
    registry.update(B200_ALGORITHMS)
    return registry
