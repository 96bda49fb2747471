#!/usr/bin/env python
"""bench.py -- QRDM2 fp64 throughput on B200 (BASELINE.json metric).

Workload at N=1: BASELINE configs[1] = cfg2, one 4096 x 4096 iid N(0,1) matrix
(seed 1, host numpy generator of paper_2106_03138_b200.inputs), factored by
qrdm2 with the reference defaults (tau 0.15, delta 0.9, k_dm 64, stop eps*n).
A "step" is one full factorization; value = nominal flops (2mn^2 - 2n^3/3) per
second.  A single matrix does not shard, so at N > 1 the headline
is cfg3: the batch of 1024 independent 256 x 256 matrices partitioned over the
ranks, with the NCCL all_gather of the per-matrix results inside the timed
region (value = matrices/s of the whole job).  The N=1 line carries cfg3 too.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config cfg2|cfg3]

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself
under torch.distributed.run with N ranks (NCCL_DEBUG=INFO).

--impl reference times the reference's own CPU implementation on the host
cores: the unmodified ``dmqr`` package installed in baseline/_ref (pip
--target) when present, else the oracle port (oracle/qrdm_oracle.py); same
config, metric and unit; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "QRDM fp64 GFLOP/s (2mn^2-2n^3/3)"
UNIT = "GFLOP/s"
METRIC3 = "QRDM matrices/s (cfg3 batch of 1024 x 256x256)"
UNIT3 = "matrices/s"
HBM_GBS = 6542.4  # MEASURED_PEAKS.json copy bandwidth (recipe value at survey time)


def nominal(m, n):
    return 2.0 * m * n * n - 2.0 * n ** 3 / 3.0


def workload_config(name: str, args, world: int) -> dict:
    """The config dict both arms print (identical by construction)."""
    if name == "cfg2":
        n = args.size
        return {"workload": f"cfg2 qrdm2 {n}x{n} N(0,1) seed {args.seed}" + (" + rank" if world > 1 else ""),
                "algo": "qrdm2", "m": n, "n": n, "tau": 0.15, "delta": 0.9, "k_dm": 64, "stop": "eps*n",
                "generator": "host numpy (paper_2106_03138_b200.inputs.cfg2)",
                "l2": "matrix (134 MB) + pristine copy exceed the 126 MB L2; each step re-copies the input"}
    return {"workload": f"cfg3 qrdm2 batch {args.batch} x 256x256 (B C + 1e-10 E) seed 3, "
                        f"sharded over {world} GPU(s)",
            "algo": "qrdm2", "batch": args.batch, "m": 256, "n": 256, "tau": 0.15, "delta": 0.9, "k_dm": 64,
            "stop": "eps*n", "generator": "host numpy (paper_2106_03138_b200.inputs.cfg3)",
            "l2": "batch (512 MiB) + pristine copy exceed the 126 MB L2; each step re-copies the inputs"}


# ----------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait()

    def summary(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------
# reference arm: the reference's CPU implementation on the host cores
# ----------------------------------------------------------------------------

def _reference_module():
    """The unmodified reference package from baseline/_ref (pip --target), or None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "dmqr" / "__init__.py").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "dmqr_numba_cache"))
    sys.path.insert(0, str(ref))
    try:
        import dmqr  # noqa: F401
        return dmqr
    except Exception as e:  # pragma: no cover -- e.g. numba missing on the box
        print(f"[bench] baseline/_ref dmqr not importable ({e}); using the oracle port", file=sys.stderr)
        sys.path.remove(str(ref))
        return None


def _cfg3_worker_init(use_ref: bool):
    global _QRDM2
    if use_ref:
        _reference_module()
        import dmqr
        _QRDM2 = dmqr.qrdm2
    else:
        from oracle import qrdm_oracle as O
        _QRDM2 = O.qrdm2


def _cfg3_worker(A):
    return int(_QRDM2(A).rank)


def cfg3_cpu_batch(B, use_ref: bool):
    """The whole cfg3 batch on every host core: multiprocessing Pool with one BLAS
    thread per worker (the drivers are pure functions, README.md:146-147;
    BASELINE.md §2).  Returns (seconds, ranks, workers)."""
    import multiprocessing as mp

    workers = len(os.sched_getaffinity(0))
    old = os.environ.get("OPENBLAS_NUM_THREADS")
    os.environ["OPENBLAS_NUM_THREADS"] = "1"  # inherited by the spawned workers
    try:
        with mp.get_context("spawn").Pool(workers, initializer=_cfg3_worker_init, initargs=(use_ref,)) as pool:
            pool.map(_cfg3_worker, [B[i] for i in range(workers)])  # warm the workers (imports, numba)
            t0 = time.perf_counter()
            ranks = pool.map(_cfg3_worker, [B[i] for i in range(B.shape[0])], chunksize=4)
            dt = time.perf_counter() - t0
    finally:
        if old is None:
            del os.environ["OPENBLAS_NUM_THREADS"]
        else:
            os.environ["OPENBLAS_NUM_THREADS"] = old
    return dt, ranks, workers


def run_reference(args, rank, world, name):
    if rank != 0:
        return
    from threadpoolctl import threadpool_info

    from paper_2106_03138_b200 import inputs

    dmqr = _reference_module()
    kind = "reference" if dmqr is not None else "port"
    impl_desc = ("dmqr.qrdm2 (unmodified reference, baseline/_ref)" if dmqr is not None
                 else "oracle/qrdm_oracle.py qrdm2 (numpy port of the reference)")
    cores = len(os.sched_getaffinity(0))
    cfg = workload_config(name, args, world)
    if name == "cfg3":
        B = inputs.cfg3(seed=3, batch=args.batch)
        times = []
        for i in range(args.warmup + args.steps):
            dt, ranks, workers = cfg3_cpu_batch(B, dmqr is not None)
            if i >= args.warmup:
                times.append(dt)
        ms = 1e3 * statistics.mean(times)
        value = args.batch / (ms / 1e3)
        unit, metric = UNIT3, METRIC3
        sample = (f"the whole {args.batch}-matrix batch per step, {impl_desc} in a multiprocessing Pool of "
                  f"{workers} workers x 1 BLAS thread")
        threads = workers
    else:
        n = args.size
        A = inputs.cfg2(seed=args.seed, n=n)
        fn = dmqr.qrdm2 if dmqr is not None else __import__("oracle.qrdm_oracle", fromlist=["x"]).qrdm2
        threads = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
        fn(A)  # warm-up (numba compilation, BLAS threads): one full factorization
        # each timed step is one full qrdm2 of the cfg2 matrix; the remaining
        # warm-ups are skipped when they would push the run past a few minutes
        t0 = time.perf_counter()
        fn(A)
        t1 = time.perf_counter() - t0
        times = [t1]
        budget = 240.0
        while len(times) < args.steps and sum(times) + t1 < budget:
            t0 = time.perf_counter()
            fn(A)
            times.append(time.perf_counter() - t0)
        ms = 1e3 * statistics.mean(times)
        value = nominal(n, n) / (ms / 1e3) / 1e9
        unit, metric = UNIT, METRIC
        sample = (f"one full qrdm2 of the cfg2 {n}x{n} matrix per step ({len(times)} timed of {args.steps} "
                  f"requested within a {budget:.0f} s budget), {impl_desc}, {threads} BLAS threads of {cores} "
                  f"host cores")
    line = {
        "impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if name == "cfg3" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": unit, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# B200 arm
# ----------------------------------------------------------------------------

def fp64_peak_tflops(torch, dev) -> float:
    """cuBLAS DGEMM 8192^3 best-of-5: the FP64 roofline denominator (not on the product path)."""
    a = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    b = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    torch.cuda.synchronize(dev)
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    del a, b
    return 2 * 8192 ** 3 / best / 1e12


def trailing_flops(m, n, steps) -> float:
    """Algorithmic flops of the trailing block update (rrqr.py:386 blocked_flops)."""
    f = 0.0
    for s in steps:
        if s.n_s + s.k_selected < n and not s.fell_back_to_scalar:
            f += (4.0 * (m - s.n_s) * s.k_accepted + 2.0 * s.k_accepted ** 2) * (n - s.n_s - s.k_selected)
    return f


def spare_flops(m, n, steps) -> list:
    """Algorithmic flops of k_spare per step (look-ahead schedule):
    phase 1 = the previous step's C -= Y Wt below its R rows (2 (m - n_s) l_prev
    n''_prev), phase 2 = G = Q1^T C (2 (m - n_s) k_s n''_s).  (Y = Q1 M runs in
    k_trail_w's extra CTAs.)"""
    out = []
    prev = None
    for s in steps:
        mp = m - s.n_s
        nn = max(n - s.n_s - s.k_selected, 0)
        f = 2.0 * mp * s.k_selected * nn
        if prev is not None:
            f += 2.0 * mp * prev.k_accepted * max(n - prev.n_s - prev.k_selected, 0)
        out.append(f)
        prev = s
    return out


def panel_bytes(m, n, steps) -> float:
    """B_panel of SURVEY §8(d) (HBM leg of the roofline), without guard recomputes."""
    b = 8.0 * m * n
    for s in steps:
        mp = m - s.n_s
        l, k = s.k_accepted, s.k_selected
        nn = n - s.n_s - k
        km = max(s.k_max, 0)
        b += 16.0 * mp * k + 8.0 * mp * (km + 1) + 8.0 * l * max(nn, 0) + 32.0 * m * k
    return b


TL_NAMES = {0: "select", 1: "gram", 2: "gram_finish", 3: "swap", 4: "panel_cq", 5: "spare", 6: "ygemm",
            7: "trail_w", 8: "trail_a", 9: "guard", 10: "step_tail", 11: "trail_b", 12: "downdate", 13: "panel_rr"}


def timeline_spans(f, m, n) -> tuple:
    """(per-step {kernel: us}, per-step step span us) from the DMQR_TIMELINE buffer
    of the factorization that ran in f's workspace (first 64 steps)."""
    import ctypes as C

    from paper_2106_03138_b200 import _lib

    tl = np.zeros(64 * 32 + 1024, dtype=np.int64)
    _lib.load().dmqr_debug_timeline(f.workspace.data_ptr(), m, n, tl.ctypes.data_as(C.c_void_p))
    t = tl[:2048].reshape(64, 16, 2).astype(np.float64)
    ok = (t[:, :, 0] > 0) & (t[:, :, 0] < 2 ** 62) & (t[:, :, 1] > 0)
    ok[:, 11:] = False  # (slots 22-27: k_trail_w's phase stamps; 28-31: k_spare's -- not spans)
    per, span = [], []
    for s in range(min(64, int(f.info.n_steps))):
        d = {TL_NAMES.get(k, str(k)): (t[s, k, 1] - t[s, k, 0]) / 1e3 for k in range(11) if ok[s, k]}
        # k_spare's busy time: phase 1 (start .. last tile done) + phase 2 (Q1 seen, after phase 1 ..
        # last G tile done); the rest of its span waits for the panel
        if ok[s, 5]:
            st0, q1_seen, p1_end, p2_end = t[s, 5, 0], t[s, 14, 0], t[s, 14, 1], t[s, 15, 1]
            busy = 0.0
            if p1_end > st0:
                busy += p1_end - st0
            if p2_end > 0 and 0 < q1_seen < 2 ** 62:
                busy += max(0.0, p2_end - max(q1_seen, p1_end, st0))
            if busy > 0:
                d["spare_busy"] = busy / 1e3
        per.append(d)
        if ok[s].any():
            span.append((t[s, ok[s], 1].max() - t[s, ok[s], 0].min()) / 1e3)
        else:
            span.append(float("nan"))
    return per, span


def load_profile_number(fname, key):
    prof = ROOT / "profiles" / fname
    if prof.exists():
        try:
            return json.loads(prof.read_text()).get(key)
        except Exception:
            return None
    return None


def other_configs(torch, dev, peak_tf):
    """BASELINE cfg4 (host-generated pinned input, parity against the reference
    golden), cfg5 16384^2 (device-generated: a host Haar QR of that size takes
    ~20 min single-threaded), qrp on cfg2: best of 2 device-timed factorizations
    each (informational; the N=1 headline stays cfg2)."""
    from paper_2106_03138_b200 import inputs, rrqr

    out = {}
    gold = None
    try:
        gold = np.load(ROOT / "tests" / "golden" / "fullsize.npz")
        gidx = json.loads((ROOT / "tests" / "golden" / "fullsize_index.json").read_text())["cases"]
    except OSError:
        gidx = {}
    for name, algo in (("cfg4", "qrdm"), ("cfg5", "qrdm"), ("cfg2_qrp", "qrp")):
        gen = "host numpy (inputs.cfg4, pinned to the reference golden)" if name == "cfg4" else \
            ("device torch RNG (inputs.device_cfg)" if name == "cfg5" else "host numpy (inputs.cfg2)")
        if name == "cfg2_qrp":
            A = inputs.cfg2(seed=1)
        elif name == "cfg4":
            A = inputs.cfg4(seed=4)
        else:
            A = inputs.device_cfg(name, seed=4)
        m, n = A.shape
        A_host = A if isinstance(A, np.ndarray) else None
        work = rrqr.to_work(A)
        del A
        b0 = work[0].clone()
        best, f = 1e30, None
        for _ in range(2):
            work[0].copy_(b0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f = rrqr.factorize(None, work=work, algo=algo)
            e1.record()
            torch.cuda.synchronize(dev)
            best = min(best, e0.elapsed_time(e1))
        steps = rrqr._steps_from_raw(f.steps.cpu().numpy(), int(f.info.n_steps))
        nf = int(f.info.n_factored)
        scal = [s for s in steps if s.fell_back_to_scalar or algo == "qrp"]
        f_dm = trailing_flops(m, n, [s for s in steps if not s.fell_back_to_scalar]) if algo != "qrp" else 0.0
        f_sc = sum(4.0 * (m - s.n_s) * (n - s.n_s - 1) for s in scal)
        b_sc = sum(8.0 * (m - s.n_s) * (n - s.n_s - 1) for s in scal)
        t_roof = (f_dm + f_sc) / (peak_tf * 1e12) * 1e3
        t_phased = (f_dm / (peak_tf * 1e12) + b_sc / (HBM_GBS * 1e9)) * 1e3
        rec = {"algo": "qrp" if algo == "qrp" else "qrdm2", "generator": gen,
               "m": m, "n": n, "ms": best, "rank": int(f.info.rank), "outer_steps": len(steps),
               "scalar_pivot_steps": sum(1 for s in steps if s.fell_back_to_scalar),
               "gflops_nominal": nominal(m, n) / (best / 1e3) / 1e9 if m >= n else None,
               "gflops_executed": (nominal(m, n) - (nominal(m - nf, n - nf) if nf < n else 0.0)) / (best / 1e3) / 1e9,
               "t_roof_ms": t_roof, "roofline_frac": t_roof / best,
               "t_roof_phased_ms": t_phased, "roofline_phased_frac": t_phased / best}
        if name == "cfg4" and gold is not None and "cfg4" in gidx:
            import hashlib
            same_in = hashlib.sha256(np.ascontiguousarray(A_host).tobytes()).hexdigest() == gidx["cfg4"]["input_sha256"]
            fwd = f.perm.cpu().numpy()
            ref = gold["cfg4/forward"].astype(np.int64)
            rec["parity_vs_reference"] = {
                "input_sha256_matches": bool(same_in), "perm_identical": bool(np.array_equal(fwd, ref)),
                "rank": int(f.info.rank), "reference_rank": int(gidx["cfg4"]["rank"]),
                "first_perm_difference": int(np.argmax(fwd != ref)) if not np.array_equal(fwd, ref) else None}
        out[name] = rec
        del work, b0, f
        torch.cuda.empty_cache()
    return out


def _time_cfg3(torch, dev, args, rank, world, with_gather: bool):
    """Device-timed cfg3 steps (copy-in of the pristine slice, batched
    factorization, NCCL all_gather of the per-matrix results) -> (ms per step,
    gathered ranks or local ranks, kernel launches, clocks)."""
    import torch.distributed as dist

    from paper_2106_03138_b200 import _lib, inputs
    from paper_2106_03138_b200.batch import factorize_batch, gather_summaries, shard, summary_tensor, to_batch_work

    B = inputs.cfg3(seed=3, batch=args.batch)
    lo, hi = shard(args.batch, rank, world)
    work0 = to_batch_work(B[lo:hi], dev)
    buf = work0[0].clone()
    work = (buf, work0[1], work0[2], work0[3])
    table = [None]

    def step():
        buf.copy_(work0[0])
        f = factorize_batch(None, lanes=args.lanes, work=work)
        if with_gather:
            table[0] = gather_summaries(summary_tensor(f, dev), args.batch)
        return f

    for _ in range(args.warmup):
        f = step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    _lib.stats(reset=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        ev0.record()
        for _ in range(args.steps):
            f = step()
        ev1.record()
        torch.cuda.synchronize(dev)
    st = _lib.stats(reset=True)
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ranks = table[0][:, 0].cpu().numpy() if with_gather else f.ranks
    return ms / args.steps, ranks, st, clk, (B, lo, hi)


def run_b200_cfg3(args, rank, world):
    """cfg3 headline (N > 1, or --config cfg3): matrices/s of the whole job with the
    NCCL gather inside the timed region."""
    import torch
    import torch.distributed as dist

    from paper_2106_03138_b200.batch import factorize_batch, gather_summaries, summary_tensor

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ms_step, ranks_all, st, clk, (B, lo, hi) = _time_cfg3(torch, dev, args, rank, world, world > 1)
    value = args.batch / (ms_step / 1e3)
    # end to end through the public batch API: pinned host slice in, gathered
    # per-matrix results (rank, n_factored, stopped, steps, perm, coeffs) out
    pinned = torch.from_numpy(np.ascontiguousarray(B[lo:hi])).pin_memory()
    e2e = []
    for i in range(args.steps + 1):
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        f = factorize_batch(pinned, lanes=args.lanes)
        tab = summary_tensor(f, dev)
        if world > 1:
            tab = gather_summaries(tab, args.batch)
        host = tab.cpu()
        e2e.append(time.perf_counter() - t0)
    e2e_s = statistics.mean(e2e[1:])
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    if rank != 0:
        return
    hist = {int(k): int(v) for k, v in zip(*np.unique(ranks_all, return_counts=True))}
    line = {
        "metric": METRIC3, "value": value, "unit": UNIT3, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload_config("cfg3", args, world),
        "run": {"lanes": args.lanes, "gflops_nominal": args.batch * nominal(256, 256) / (ms_step / 1e3) / 1e9,
                "rank_histogram": hist, "collective": "all_gather_into_tensor (NCCL) of the per-matrix results "
                                                      "inside the timed region" if world > 1 else "none (N=1)"},
        "gpu_launches": int(st["kernel_launches"]),
        "e2e": {"value": args.batch / e2e_s, "unit": UNIT3, "h2d_bytes_per_step": int(8 * 256 * 256 * (hi - lo)),
                "d2h_bytes_per_step": int(host.numel() * host.element_size()), "ms_per_step": 1e3 * e2e_s,
                "path": "batch.factorize_batch(pinned host slice) + summary_tensor + all_gather -> host"},
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def run_b200(args, rank, world):
    import torch
    import torch.distributed as dist

    from paper_2106_03138_b200 import _lib, inputs, rrqr

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n = args.size
    A = inputs.cfg2(seed=args.seed + rank, n=n)
    lib = _lib.load()

    work0 = rrqr.to_work(A, dev)
    buf0 = work0[0]
    buf = buf0.clone()
    work = (buf, work0[1], work0[2], work0[3])

    def step():
        buf.copy_(buf0)
        return rrqr.factorize(None, rrqr.DMParams(), rrqr.StopCriterion(), break_check=True, work=work)

    for _ in range(args.warmup):
        f = step()
    torch.cuda.synchronize(dev)
    last = rrqr.to_result(f)
    steps_log = last.step_log

    peak_tf = fp64_peak_tflops(torch, dev)
    if world > 1:
        dist.barrier()
    _lib.stats(reset=True)
    torch.cuda.synchronize(dev)
    # the timed region runs the production schedule (no phase events); the last
    # timed factorization also records the per-kernel device timeline
    # (DMQR_TIMELINE: one globaltimer stamp pair per kernel and step, taken with
    # atomics by thread 0 of each CTA), which the roofline block reads
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        ev0.record()
        for i in range(args.steps):
            if i == args.steps - 1:
                os.environ["DMQR_TIMELINE"] = "1"
            f = step()
        ev1.record()
        torch.cuda.synchronize(dev)
    os.environ.pop("DMQR_TIMELINE", None)
    st = _lib.stats(reset=True)
    ms = ev0.elapsed_time(ev1)
    per_kernel, step_span = timeline_spans(f, n, n)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    ms_step = ms / args.steps
    value = world * nominal(n, n) / (ms_step / 1e3) / 1e9

    # ---- phase split (separate pass: per-step event records serialize the launches) ----
    lib.dmqr_stats_enable(1)
    _lib.stats(reset=True)
    step()
    torch.cuda.synchronize(dev)
    phases = _lib.stats(reset=True)
    lib.dmqr_stats_enable(0)

    # ---- end to end through the public API, host buffers in and out ----
    pinned = torch.from_numpy(np.ascontiguousarray(A)).pin_memory()
    e2e_ms = []
    res = None
    for i in range(args.steps + 2):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        res = rrqr.qrdm2(pinned)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = e2e_ms[2:]  # first two calls populate the device and pinned-host caches
    e2e_step = statistics.mean(e2e_ms)
    h2d = 8 * n * n
    d2h = 8 * n * n + 8 * n + 8 * n + 16 * len(res.perm.swaps) + 56 * len(res.step_log)
    e2e_val = world * nominal(n, n) / (e2e_step / 1e3) / 1e9
    if world > 1:
        t = torch.tensor([e2e_step], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_val = world * nominal(n, n) / (float(t.item()) / 1e3) / 1e9

    # ---- roofline: k_spare (the look-ahead schedule's dense contraction) from
    # the timed run's device timeline; the step roofline of SURVEY §8(d) ----
    ftr = trailing_flops(n, n, steps_log)
    fsp = spare_flops(n, n, steps_log)
    sp_us = [d.get("spare") for d in per_kernel]
    pairs = [(fl, us) for fl, us in zip(fsp, sp_us) if us]
    achieved = (sum(fl for fl, _ in pairs) / (sum(us for _, us in pairs) / 1e6) / 1e12) if pairs else None
    bpairs = [(fl, d.get("spare_busy")) for fl, d in zip(fsp, per_kernel) if d.get("spare_busy")]
    achieved_busy = (sum(fl for fl, _ in bpairs) / (sum(us for _, us in bpairs) / 1e6) / 1e12) if bpairs else None
    step_sum = {}
    for d in per_kernel:
        for k, v in d.items():
            step_sum[k] = step_sum.get(k, 0.0) + v
    span_ms = float(np.nansum(step_span)) / 1e3
    bp = panel_bytes(n, n, steps_log)
    t_roof_ms = max(ftr / (peak_tf * 1e12), bp / (HBM_GBS * 1e9)) * 1e3

    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        from threadpoolctl import threadpool_info

        from oracle import qrdm_oracle as O  # the checker / baseline only

        dmqr_ref = _reference_module()  # the unmodified reference when baseline/_ref travelled, else the port
        t0 = time.perf_counter()
        if dmqr_ref is not None:
            ref = dmqr_ref.qrdm2(A)
            ref_fwd, ref_rank = np.asarray(ref.perm.forward), int(ref.rank)
        else:
            ref = O.qrdm2(A)
            ref_fwd, ref_rank = ref.forward, ref.rank
        t_cpu = time.perf_counter() - t0
        threads = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
        same = bool(np.array_equal(ref_fwd, last.perm.forward)) and ref_rank == last.rank
        who = ("the unmodified reference dmqr.qrdm2 (baseline/_ref)" if dmqr_ref is not None
               else "the numpy oracle port (oracle/qrdm_oracle.py)")
        cpu = {"value": nominal(n, n) / t_cpu / 1e9, "unit": UNIT, "cores": threads,
               "kind": "reference" if dmqr_ref is not None else "port",
               "sample": f"one full qrdm2 of the same cfg2 {n}x{n} matrix ({t_cpu:.1f} s) with {who}, "
                         f"{threads} BLAS threads of {len(os.sched_getaffinity(0))} host cores; "
                         f"GPU perm/rank identical: {same}"}
    extra = None
    if world == 1 and not args.no_extra:
        extra = other_configs(torch, dev, peak_tf)
        ms3, ranks3, st3, _, (B3, _, _) = _time_cfg3(torch, dev, args, 0, 1, False)
        c3 = {"algo": "qrdm2", "batch": args.batch, "m": 256, "n": 256, "ms": ms3,
              "matrices_per_s": args.batch / (ms3 / 1e3),
              "gflops_nominal": args.batch * nominal(256, 256) / (ms3 / 1e3) / 1e9,
              "rank_histogram": {int(k): int(v) for k, v in zip(*np.unique(ranks3, return_counts=True))}}
        if not args.no_cpu:
            from paper_2106_03138_b200 import inputs as _in  # noqa: F401
            dt, r_cpu, workers = cfg3_cpu_batch(B3, _reference_module() is not None)
            c3["cpu_baseline"] = {"value": args.batch / dt, "unit": UNIT3, "cores": workers,
                                  "kind": "reference" if _reference_module() is not None else "port",
                                  "sample": f"all {args.batch} matrices, multiprocessing Pool of {workers} "
                                            f"workers x 1 BLAS thread ({dt:.2f} s)",
                                  "rank_histogram": {int(k): int(v) for k, v in
                                                     zip(*np.unique(r_cpu, return_counts=True))}}
        extra["cfg3"] = c3
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload_config("cfg2", args, world),
        "run": {"rank": last.rank, "outer_steps": len(steps_log)},
        "gpu_launches": int(st["kernel_launches"]),
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e2e_step, "path": "paper_2106_03138_b200.qrdm2(pinned host tensor) -> numpy result"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": (achieved / peak_tf) if achieved else None,
                     "traffic": load_profile_number("r02_spare_traffic.json", "traffic_bytes_per_launch"),
                     "kernel": "k_spare (persistent, beside the panel: previous step's C -= Y Wt, then G = Q1^T C "
                               "once the panel has published Q1; DMMA m8n8k4 f64), spans from the timed run's "
                               "device timeline (last timed factorization)",
                     "achieved_busy": achieved_busy,
                     "frac_busy": (achieved_busy / peak_tf) if achieved_busy else None,
                     "busy_note": "achieved/frac are over k_spare's whole spans, which include its wait for the "
                                  "panel's Q1; *_busy count only the time between its first tile and the last "
                                  "tile of each phase (phase stamps of the same timeline)",
                     "algorithmic_flops_per_factorization": sum(fsp),
                     "spare_us_per_factorization": sum(us for _, us in pairs),
                     "peak_source": "cuBLAS DGEMM 8192^3 best-of-5 measured in this run (FP64 peak; "
                                    "MEASURED_PEAKS.json has bf16 only)"},
        "step_roofline": {"t_roof_ms": t_roof_ms, "t_step_ms": ms_step, "frac": t_roof_ms / ms_step,
                          "trailing_flops": ftr, "panel_bytes": bp, "hbm_gbs": HBM_GBS},
        "timeline_us_per_factorization": {k: round(v, 1) for k, v in sorted(step_sum.items(), key=lambda x: -x[1])},
        "timeline_note": "device spans (first CTA start to last CTA exit) summed over the steps of the last "
                         f"timed factorization; step spans sum to {span_ms:.2f} ms",
        "phases_ms_per_step": {k: phases[k] for k in ("ms_select", "ms_panel", "ms_trailing", "ms_norms")},
        "phases_note": "one extra factorization with per-step phase events (serializes the programmatic "
                       "launches at phase boundaries); ms_panel includes k_spare",
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "other_configs": extra,
    }
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_distributed(n: int) -> int:
    """Re-run this script under torch.distributed.run with n ranks (one per GPU)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the cfg3 / cfg4 / cfg5 / qrp information block")
    ap.add_argument("--config", default=None, choices=["cfg2", "cfg3"],
                    help="headline workload (default: cfg2 at N=1, cfg3 at N>1)")
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--lanes", type=int, default=4)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args.gpus))
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    name = args.config or ("cfg2" if world == 1 else "cfg3")
    if world > 1:
        import torch.distributed as dist
        if args.impl == "b200":
            import torch
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
            dist.init_process_group("nccl")
        else:
            dist.init_process_group("gloo")
    if args.impl == "reference":
        run_reference(args, rank, world, name)
    elif name == "cfg3":
        run_b200_cfg3(args, rank, world)
    else:
        run_b200(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
