"""Drop-in QRDM / QRDM2 drivers backed by the B200 kernels.

Same call and result surface as the reference ``dmqr.rrqr`` (rrqr.py:39-53,
426-456) and ``dmqr.dm.DMParams`` (dm.py:41-62):

    qrdm (A, params=DMParams(), stop=StopCriterion(), trace_norms=False) -> RRQRResult
    qrdm2(A, params=DMParams(), stop=StopCriterion(), trace_norms=False) -> RRQRResult
    qrp  (A, stop=StopCriterion(), trace_norms=False) -> RRQRResult   (rrqr.py:238-291)

The factorization itself runs in ``libdmqr_b200.so`` (hand-written sm_100a
CUDA, called through the C-ABI in include/dmqr_b200.h).  PyTorch only carries
device buffers and the stream.  There is no CPU fallback: without a CUDA
device or the built library these functions raise.

Differences from the reference that are by design:
  * ``packed``/``coeffs`` come back as numpy arrays by default (as in the
    reference); ``device=True`` keeps them as torch CUDA tensors.
  * any k_dm >= 1 is accepted (dm.py:56-62); above 64 the engine selects with
    the wide kernels (csrc/wide.cuh) and runs a step's block as panel chunks.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib

EPS = float(np.finfo(np.float64).eps)
K_DM_FAST = 64  # k_dm above this: wide selection kernels (csrc/wide.cuh)


def engine_k_dm(k_dm: int, n: int) -> int:
    """k_dm as the engine takes it: at most n - 1 candidates exist besides the
    seed, so min(k_dm, n - 1) selects exactly what k_dm does (dm.py:95-97)."""
    return int(max(1, min(int(k_dm), max(n - 1, 1))))


def swap_capacity(kmax: int, k_dm: int) -> int:
    """Swap-log capacity: at most k_s <= k_dm + 1 transpositions per step
    (rrqr.py:294-312); very wide selections are capped at 2^24 entries (the
    engine reports DMQR_ECAP past it)."""
    cap = max(kmax * (k_dm + 1) + 8, 8)
    return cap if k_dm <= K_DM_FAST else max(kmax * (K_DM_FAST + 1) + 8, min(cap, 1 << 24))

__all__ = [
    "EPS", "DMParams", "StopRule", "StopCriterion", "StepRecord", "WorkCounters", "Permutation",
    "RRQRResult", "qrdm", "qrdm2", "qrp", "reconstruct", "factorize",
]


# ----------------------------------------------------------------------------
# parameter / result types (mirrors of dm.py:41-78 and rrqr.py:58-158)
# ----------------------------------------------------------------------------

@dataclass(frozen=True)
class DMParams:
    """tau in (0, 1], delta in [0, 1), k_dm >= 1 -- dm.py:41-62 (same messages)."""

    tau: float = 0.15
    delta: float = 0.9
    k_dm: int = 64
    use_delta_max: bool = False

    def __post_init__(self):
        if not 0.0 < self.tau <= 1.0:
            raise ValueError(f"tau must be in (0, 1], got {self.tau}")
        if not 0.0 <= self.delta < 1.0:
            raise ValueError(f"delta must be in [0, 1), got {self.delta}")
        if self.k_dm < 1:
            raise ValueError(f"k_dm must be >= 1, got {self.k_dm}")


class StopRule(Enum):
    EPS_N = "n"
    EPS_SQRT_N = "sqrt-n"
    NONE = "none"


_RULE_CODE = {StopRule.EPS_N: 0, StopRule.EPS_SQRT_N: 1, StopRule.NONE: 2}


def rule_code(stop) -> int:
    """C-ABI stop_rule code of a StopCriterion -- ours or the reference's own
    (rrqr.py:58-80): the reference harness passes dmqr.rrqr.StopCriterion
    objects, whose StopRule enum is keyed by the same values."""
    return {"n": 0, "sqrt-n": 1, "none": 2}[StopRule(getattr(stop.variant, "value", stop.variant)).value]


@dataclass(frozen=True)
class StopCriterion:
    variant: StopRule = StopRule.EPS_N
    epsilon: float = EPS

    @classmethod
    def from_name(cls, name: str) -> "StopCriterion":
        return cls(StopRule(name))

    def eps1(self, n: int):
        if self.variant is StopRule.EPS_N:
            return self.epsilon * n
        if self.variant is StopRule.EPS_SQRT_N:
            return self.epsilon * math.sqrt(n)
        return None


@dataclass
class StepRecord:
    n_s: int
    k_selected: int
    k_accepted: int
    broke_early: bool = False
    fell_back_to_scalar: bool = False
    eps_s: float = 0.0
    gamma: float = 1.0
    k_max: int = -1  # extra: candidate-set size (not in the reference record)


@dataclass
class WorkCounters:
    rank1_flops: float = 0.0
    blocked_flops: float = 0.0
    total_flops: float = 0.0

    @property
    def rank1_fraction(self) -> float:
        return self.rank1_flops / self.total_flops if self.total_flops else 0.0

    @property
    def blocked_fraction(self) -> float:
        return self.blocked_flops / self.total_flops if self.total_flops else 0.0


class Permutation:
    """forward map + swap log (matrix.py:90-152)."""

    def __init__(self, n: int):
        self.forward = np.arange(n, dtype=np.intp)
        self._swaps: list | None = []
        self._swap_rows = None  # (count, 2) integer array from the device log, listed on first use

    @property
    def swaps(self) -> list:
        """The transposition log as the reference's list of (i, j) tuples; the
        device log arrives as one array and is listed when first read."""
        if self._swaps is None:
            self._swaps = list(map(tuple, self._swap_rows.tolist()))
        return self._swaps

    @swaps.setter
    def swaps(self, value) -> None:
        self._swaps, self._swap_rows = list(value), None

    def set_swap_rows(self, rows: np.ndarray) -> None:
        self._swaps, self._swap_rows = None, rows

    @property
    def n(self) -> int:
        return int(self.forward.size)

    def replay(self) -> np.ndarray:
        fwd = np.arange(self.n, dtype=np.intp)
        for i, j in self.swaps:
            fwd[i], fwd[j] = fwd[j], fwd[i]
        return fwd

    def inverse(self) -> np.ndarray:
        inv = np.empty(self.n, dtype=np.intp)
        inv[self.forward] = np.arange(self.n, dtype=np.intp)
        return inv

    def __eq__(self, other) -> bool:
        return isinstance(other, Permutation) and np.array_equal(self.forward, other.forward)

    def __repr__(self) -> str:
        return f"Permutation({list(self.forward)})"


@dataclass
class RRQRResult:
    packed: object
    coeffs: object
    perm: Permutation
    rank: int
    step_log: list
    n_factored: int
    stopped_early: bool
    counters: WorkCounters = field(default_factory=WorkCounters)
    norm_trace: list = field(default_factory=list)
    device_time_ms: float | None = None

    @property
    def m(self) -> int:
        return int(self.packed.shape[0])

    @property
    def n(self) -> int:
        return int(self.packed.shape[1])

    def r_diagonal(self):
        d = self.packed.diagonal()[: self.n_factored]
        return d.copy() if isinstance(d, np.ndarray) else d.clone()


# ----------------------------------------------------------------------------
# counters replay (rrqr.py:330,356,366-373,384-391,230-235,346) -- SURVEY App. C
# ----------------------------------------------------------------------------

class LazyCounters:
    """WorkCounters replayed from the step log on first access (the replay is a
    Python loop over every accepted column; most callers never read it)."""

    def __init__(self, m: int, n: int, steps: list, qrp: bool = False):
        self._args = (m, n, steps, qrp)
        self._wc = None

    def _get(self) -> WorkCounters:
        if self._wc is None:
            self._wc = replay_counters(*self._args)
        return self._wc

    def __getattr__(self, name):
        if name.startswith("_"):
            raise AttributeError(name)
        return getattr(self._get(), name)

    def __eq__(self, other):
        return self._get() == (other._get() if isinstance(other, LazyCounters) else other)

    def __repr__(self):
        return repr(self._get())


def replay_counters(m: int, n: int, steps: list, qrp: bool = False) -> WorkCounters:
    """qrp: every step is one _scalar_step + downdate (rrqr.py:230-235, 275)."""
    wc = WorkCounters(total_flops=2.0 * m * n)
    for st in steps:
        s = st.n_s
        if st.fell_back_to_scalar or qrp:
            if s + 1 < n:
                f = 4.0 * (m - s) * (n - s - 1)
                wc.rank1_flops += f
                wc.total_flops += f
            wc.total_flops += 4.0 * (m - s) + (n - s)
            wc.total_flops += 4.0 * (n - s - 1)
            continue
        k_s, l = st.k_selected, st.k_accepted
        wc.total_flops += (m - s) * (st.k_max + 1) ** 2
        for col in range(s, s + l):
            if col + 1 < s + k_s:
                f = 4.0 * (m - col) * (s + k_s - col - 1)
                wc.rank1_flops += f
                wc.total_flops += f
            wc.total_flops += 4.0 * (m - col)
        if s + k_s < n:
            wc.total_flops += 2.0 * (m - s) * l ** 2
            f = (4.0 * (m - s) * l + 2.0 * l ** 2) * (n - s - k_s)
            wc.blocked_flops += f
            wc.total_flops += f
        s1 = s + l
        wc.total_flops += 2.0 * l * (n - s1) if s1 < n else 0.0
    return wc


# ----------------------------------------------------------------------------
# device plumbing
# ----------------------------------------------------------------------------

def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2106_03138_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _check(rc: int):
    if rc == 0:
        return
    msg = _lib.strerror(rc)
    if rc in (_lib.DMQR_EINVAL, _lib.DMQR_ENONFINITE, _lib.DMQR_EZEROCOL):
        raise ValueError(msg)
    raise RuntimeError(f"dmqr_b200: {msg} (code {rc})")


def lda_for(m: int) -> int:
    """Leading dimension: rows rounded up to 8 doubles (64-byte aligned columns)."""
    return max(8, (m + 7) // 8 * 8)


def to_work(A, device=None):
    """Validated column-major float64 device copy of A (dense(), matrix.py:24-34).

    Returns (buf, m, n, lda) where ``buf`` is an (n, lda) torch tensor whose
    row j is column j of the matrix.
    """
    torch = _torch()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if isinstance(A, torch.Tensor):
        t = A.detach()
        if t.dim() != 2:
            raise ValueError(f"expected a 2-d array, got ndim={t.dim()}")
        t = t.to(device=dev, dtype=torch.float64)
    else:
        a = np.asarray(A, dtype=np.float64)
        if a.ndim != 2:
            raise ValueError(f"expected a 2-d array, got ndim={a.ndim}")
        t = torch.from_numpy(np.ascontiguousarray(a.T)).to(dev, non_blocking=False).T
    m, n = int(t.shape[0]), int(t.shape[1])
    lda = lda_for(m)
    # (rows m..lda of every column are padding the kernels may read: zero them unless there are none)
    alloc = torch.empty if (lda == m and n) else torch.zeros
    buf = alloc((max(n, 1), lda), dtype=torch.float64, device=dev)
    if m and n:
        buf[:n, :m].copy_(t.T)
    return buf, m, n, lda


@dataclass
class DeviceFactor:
    """Raw device outputs of one factorization (no host copies)."""

    buf: object          # (n, lda) torch tensor, column-major packed factor
    m: int
    n: int
    lda: int
    coeffs: object       # torch (kmax,)
    perm: object         # torch int64 (n,)
    swaps: object        # torch int64 (cap, 2)
    steps: object        # torch uint8 raw records
    norm_trace: object
    info: _lib.Info
    workspace: object = None
    host_packed: object = None  # pinned (n, m) host copy streamed by the engine, if requested
    algo: str = "qrdm"          # "qrp": greedy column pivoting (counters replay differs)

    def debug_ctl(self) -> dict:
        """Decision state of the last step (debug aid)."""
        import torch
        out = torch.zeros(16 + 4 * 72 + 5, dtype=torch.int64, device=self.buf.device)
        _check(_lib.load().dmqr_debug_ctl(self.workspace.data_ptr(), out.data_ptr(),
                                          C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        v = out.cpu().numpy()
        keys = ["n_s", "done", "stopped", "status", "kind", "k_max", "ncand", "nsel", "k_s", "l_acc", "nsw",
                "step_idx", "n_swaps"]
        d = {k: int(v[i]) for i, k in enumerate(keys)}
        for i, k in enumerate(["umax", "eps_s", "gamma"]):
            d[k] = float(v[13 + i:14 + i].view(np.float64)[0])
        d["cand"], d["sel"] = v[16:88].tolist(), v[88:160].tolist()
        d["sw_a"], d["sw_b"] = v[160:232].tolist(), v[232:304].tolist()
        d["cq_diag"] = v[304:308].view(np.float64).tolist()
        d["cq_fail"], d["tc0"] = int(v[308]) // 1000000, int(v[308]) % 1000000
        return d


def factorize(A, params: DMParams = DMParams(), stop: StopCriterion = StopCriterion(),
              break_check: bool = True, trace_norms: bool = False, stream=None, work=None,
              max_steps: int = 0, host_packed=None, algo: str = "qrdm") -> DeviceFactor:
    """Run one factorization on the device; returns device buffers.

    ``work`` may be a (buf, m, n, lda) tuple from ``to_work`` whose buffer is
    factored in place (the benchmark uses this to keep inputs resident).
    """
    torch = _torch()
    lib = _lib.load()
    buf, m, n, lda = work if work is not None else to_work(A)
    k_dm = engine_k_dm(params.k_dm, n)
    dev = buf.device
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    sh = C.c_void_p(st.cuda_stream)
    p = _lib.Params(tau=float(params.tau), delta=float(params.delta), epsilon=float(stop.epsilon),
                    k_dm=k_dm, use_delta_max=int(bool(params.use_delta_max)),
                    stop_rule=rule_code(stop), break_check=int(bool(break_check)),
                    trace_norms=int(bool(trace_norms)), max_steps=int(max_steps))
    kmax = min(m, n)
    step_cap = max(kmax, 1)
    swap_cap = swap_capacity(kmax, k_dm)
    coeffs = torch.zeros(max(kmax, 1), dtype=torch.float64, device=dev)
    perm = torch.arange(max(n, 1), dtype=torch.int64, device=dev)
    swaps = torch.empty((swap_cap, 2), dtype=torch.int64, device=dev)
    steps = torch.empty(step_cap * _lib.STEP_BYTES, dtype=torch.uint8, device=dev)
    ntrace = torch.full((step_cap,), float("nan"), dtype=torch.float64, device=dev) if trace_norms else None
    wsb = int(lib.dmqr_workspace_bytes(m, n, C.byref(p)))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    info = _lib.Info()
    # host_packed: pinned (n, m) host tensor; the engine streams the finished
    # columns of the packed factor into it while it runs
    hp = host_packed.data_ptr() if host_packed is not None else None
    entry = lib.dmqr_qrp_stream_f64 if algo == "qrp" else lib.dmqr_qrdm_stream_f64
    rc = entry(buf.data_ptr(), m, n, lda, C.byref(p), coeffs.data_ptr(), perm.data_ptr(),
                                  swaps.data_ptr(), swap_cap, steps.data_ptr(), step_cap,
                                  ntrace.data_ptr() if ntrace is not None else None, ws.data_ptr(), wsb,
                                  C.byref(info), hp, m, sh)
    _check(rc)
    return DeviceFactor(buf, m, n, lda, coeffs[:kmax], perm[:n], swaps, steps, ntrace, info, ws, host_packed, algo)


def _steps_from_raw(raw: np.ndarray, count: int) -> list:
    recs = np.frombuffer(raw[: count * _lib.STEP_BYTES].tobytes(), dtype=np.dtype([
        ("n_s", "<i8"), ("k_selected", "<i8"), ("k_accepted", "<i8"), ("k_max", "<i8"),
        ("broke_early", "<i4"), ("fell_back_to_scalar", "<i4"), ("eps_s", "<f8"), ("gamma", "<f8")]))
    return [StepRecord(int(r["n_s"]), int(r["k_selected"]), int(r["k_accepted"]), bool(r["broke_early"]),
                       bool(r["fell_back_to_scalar"]), float(r["eps_s"]), float(r["gamma"]), int(r["k_max"]))
            for r in recs]


def _pinned_copy(t):
    """Host copy of device tensor ``t`` in page-locked memory (the returned numpy
    view keeps the block alive; freed blocks are recycled by torch's allocator)."""
    torch = _torch()
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t)
    return out


def _fetch(tensors: list) -> list:
    """Host numpy copies of several small device tensors: asynchronous copies
    into one page-locked block, one stream synchronization."""
    torch = _torch()
    sizes = [t.numel() * t.element_size() for t in tensors]
    offs = np.concatenate([[0], np.cumsum([(b + 15) // 16 * 16 for b in sizes])]).tolist()
    host = torch.empty(max(int(offs[-1]), 16), dtype=torch.uint8, pin_memory=True)
    views = []
    for t, b, o in zip(tensors, sizes, offs):
        hv = host[o:o + b].view(t.dtype).view(t.shape)
        if b:
            hv.copy_(t, non_blocking=True)
        views.append(hv)
    torch.cuda.current_stream(tensors[0].device).synchronize()
    return [v.numpy() for v in views]


def to_result(f: DeviceFactor, device: bool = False) -> RRQRResult:
    info = f.info
    packed_t = f.buf[: f.n, : f.m].T  # m x n view
    nst, nsw = int(info.n_steps), int(info.n_swaps)
    want = [f.steps[: nst * _lib.STEP_BYTES], f.perm, f.swaps[:nsw].contiguous()]
    host_coeffs = not device and f.m and f.n
    if host_coeffs:
        want.append(f.coeffs)
    if f.norm_trace is not None:
        want.append(f.norm_trace[:nst])
    got = _fetch(want)
    steps = _steps_from_raw(got[0], nst)
    perm = Permutation(f.n)
    perm.forward = got[1].astype(np.intp, copy=False)
    perm.set_swap_rows(got[2])
    trace = []
    if f.norm_trace is not None:
        trace = [float(x) for x in got[-1] if not np.isnan(x)]
    if device:
        packed, coeffs = packed_t, f.coeffs
    elif f.m and f.n:
        # rows of buf are the columns: an (n, m) row-major host copy viewed as an
        # F-ordered (m, n) -- streamed by the engine during the factorization when
        # a pinned buffer was passed, else copied now into page-locked memory
        # (a pageable copy of a 4096^2 factor runs at ~2 GB/s, a pinned one at ~55)
        hp = f.host_packed
        packed = (hp if hp is not None else _pinned_copy(f.buf[: f.n, : f.m])).numpy().T
        coeffs = got[3]
    else:
        packed, coeffs = np.zeros((f.m, f.n), order="F"), np.zeros(0)
    return RRQRResult(packed=packed, coeffs=coeffs, perm=perm, rank=int(info.rank), step_log=steps,
                      n_factored=int(info.n_factored), stopped_early=bool(info.stopped_early),
                      counters=LazyCounters(f.m, f.n, steps, f.algo == "qrp"),
                      norm_trace=trace)


def _run(A, params, stop, break_check, trace_norms, device, algo="qrdm") -> RRQRResult:
    torch = _torch()
    work = to_work(A)
    hp = None
    if not device and work[1] and work[2]:
        hp = torch.empty((work[2], work[1]), dtype=torch.float64, pin_memory=True)
    return to_result(factorize(None, params, stop, break_check=break_check, trace_norms=trace_norms, work=work,
                               host_packed=hp, algo=algo), device)


def qrdm(A, params: DMParams = DMParams(), stop: StopCriterion = StopCriterion(),
         trace_norms: bool = False, device: bool = False) -> RRQRResult:
    """Blocked QR with deviation-maximization pivoting (rrqr.py:426-440), on the B200."""
    return _run(A, params, stop, False, trace_norms, device)


def qrdm2(A, params: DMParams = DMParams(), stop: StopCriterion = StopCriterion(),
          trace_norms: bool = False, device: bool = False) -> RRQRResult:
    """``qrdm`` plus the within-block break check (rrqr.py:443-456), on the B200."""
    return _run(A, params, stop, True, trace_norms, device)


def qrp(A, stop: StopCriterion = StopCriterion(), trace_norms: bool = False,
        device: bool = False) -> RRQRResult:
    """QR with greedy column pivoting (rrqr.py:238-291), on the B200.

    The pivot at step s is the trailing column of maximum partial norm (ties
    to the smallest index); with an active stop rule the factorization halts
    once the trailing block is negligible and rank = steps done, with
    StopRule.NONE it runs to completion and counts |r_ii| > eps n max|a_j|.
    Runs on the blocked scalar-pivot engine (delayed block updates)."""
    return _run(A, DMParams(), stop, False, trace_norms, device, algo="qrp")


def form_q(packed, coeffs, n_factored: int, qcols: int | None = None):
    """Explicit Q (m x qcols, default m) on the device (rrqr.py:468-476)."""
    torch = _torch()
    lib = _lib.load()
    P = packed if isinstance(packed, torch.Tensor) else torch.as_tensor(np.asarray(packed, dtype=np.float64))
    P = P.to("cuda", torch.float64)
    m, n = int(P.shape[0]), int(P.shape[1])
    qcols = m if qcols is None else int(qcols)
    lda = lda_for(m)
    pbuf = torch.zeros((max(n, 1), lda), dtype=torch.float64, device=P.device)
    pbuf[:n, :m].copy_(P.T)
    cf = coeffs if isinstance(coeffs, torch.Tensor) else torch.as_tensor(np.asarray(coeffs, dtype=np.float64))
    cf = cf.to(P.device, torch.float64).contiguous()
    if cf.numel() == 0:
        cf = torch.zeros(1, dtype=torch.float64, device=P.device)
    qbuf = torch.empty((max(qcols, 1), lda), dtype=torch.float64, device=P.device)
    wsb = int(lib.dmqr_form_q_workspace_bytes(m, qcols))
    ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=P.device)
    sh = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _check(lib.dmqr_form_q_f64(pbuf.data_ptr(), m, n, lda, cf.data_ptr(), int(n_factored), qbuf.data_ptr(),
                               qcols, lda, ws.data_ptr(), wsb, sh))
    return qbuf[:qcols, :m].T


def reconstruct(result: RRQRResult):
    """(Q, R) with Q m x m orthogonal and Q @ R == A @ Pi (rrqr.py:459-480); Q formed on the device."""
    Q = form_q(result.packed, result.coeffs, result.n_factored)
    Q = Q.cpu().numpy()
    packed = result.packed if isinstance(result.packed, np.ndarray) else result.packed.cpu().numpy()
    R = np.asfortranarray(np.array(packed, copy=True))
    for j in range(min(result.n_factored, R.shape[1])):
        R[j + 1:, j] = 0.0
    return np.asfortranarray(Q), R
