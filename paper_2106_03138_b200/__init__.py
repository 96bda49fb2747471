"""B200-native QRDM / QRDM2 (Deviation-Maximization rank-revealing QR, arXiv 2106.03138).

Drop-in for the reference package's hot path (``dmqr.qrdm`` / ``dmqr.qrdm2``, and ``dmqr.qrp`` on the
same scalar-pivot engine that runs QRDM's fallback steps).
The factorization runs in hand-written sm_100a CUDA (``libdmqr_b200.so``,
C-ABI in ``include/dmqr_b200.h``); there is no CPU fallback.
"""

from .rrqr import (  # noqa: F401
    EPS,
    DMParams,
    Permutation,
    RRQRResult,
    StepRecord,
    StopCriterion,
    StopRule,
    WorkCounters,
    factorize,
    form_q,
    qrdm,
    qrdm2,
    qrp,
    reconstruct,
    replay_counters,
)

__version__ = "0.1.0"
