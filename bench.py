#!/usr/bin/env python
"""bench.py -- QRDM2 fp64 throughput on B200 (BASELINE.json metric).

Workload (N=1): BASELINE configs[1] = cfg2, one 4096 x 4096 iid N(0,1) matrix
(seed 1, host numpy generator of paper_2106_03138_b200.inputs), factored by
qrdm2 with the reference defaults (tau 0.15, delta 0.9, k_dm 64, stop eps*n).
A "step" is one full factorization.  value = nominal flops (2mn^2 - 2n^3/3)
per second, whole job.  With N > 1 every rank factors its own independent
matrix (seed 1 + rank): weak scaling, no data-path collective.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--impl reference times the reference algorithm's CPU implementation on the
host cores (the oracle port in oracle/, with all BLAS threads), on the same
config; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "QRDM fp64 GFLOP/s (2mn^2-2n^3/3)"
UNIT = "GFLOP/s"


def nominal(m, n):
    return 2.0 * m * n * n - 2.0 * n ** 3 / 3.0


def partial_nominal(m, n, c):
    """Nominal flops of the first c columns of an m x n QR."""
    return nominal(m, n) - (nominal(m - c, n - c) if c < n else 0.0)


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
# reference arm: the CPU algorithm (oracle port) on the host cores
# ----------------------------------------------------------------------------

def run_reference(args, rank, world):
    if rank != 0:
        return
    from threadpoolctl import threadpool_info

    from oracle import qrdm_oracle as O
    from paper_2106_03138_b200 import inputs

    n = args.size
    A = inputs.cfg2(seed=args.seed, n=n)
    cores = len(os.sched_getaffinity(0))
    threads = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    budget_s = 200.0
    t0 = time.perf_counter()
    full = O.qrdm2(A)  # first warm-up step: the full factorization
    t_full = time.perf_counter() - t0
    S = 0  # all steps
    nsteps_full = len(full.steps)
    remaining = args.steps + max(args.warmup - 1, 0)
    if remaining * t_full > budget_s:
        frac = budget_s / (remaining * t_full)
        S = max(1, int(nsteps_full * frac))
    for _ in range(max(args.warmup - 1, 0)):
        O.qrdm2(A, max_steps=S)
    times = []
    cols = full.n_factored
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = O.qrdm2(A, max_steps=S)
        times.append(time.perf_counter() - t0)
        cols = r.n_factored if S else full.n_factored
    flops = nominal(n, n) if not S else partial_nominal(n, n, sum(s.k_accepted for s in r.steps))
    tot = sum(times)
    value = flops * len(times) / tot / 1e9
    sample = (f"full qrdm2 of the cfg2 {n}x{n} matrix per step" if not S else
              f"first {S} of {nsteps_full} outer steps ({cols} columns) of the cfg2 {n}x{n} qrdm2 per step "
              f"(full run {t_full:.1f} s); flops = nominal flops of those columns")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": f"cfg2 qrdm2 {n}x{n} N(0,1) seed {args.seed}",
                                         "algo": "qrdm2", "m": n, "n": n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample + f"; oracle/qrdm_oracle.py (numpy/OpenBLAS, {threads} threads "
                                            f"of {cores} host cores)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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
        if s.n_s + s.k_selected < n:
            f += (4.0 * (m - s.n_s) * s.k_accepted + 2.0 * s.k_accepted ** 2) * (n - s.n_s - s.k_selected)
    return f


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


def other_configs(torch, dev, peak_tf):
    """BASELINE cfg4 / cfg5 (device-generated inputs, tools/cfg_timing.py recipe) and
    qrp on cfg2: best of 2 device-timed factorizations each (informational; the
    headline stays cfg2)."""
    from paper_2106_03138_b200 import inputs, rrqr

    out = {}
    for name, algo in (("cfg4", "qrdm"), ("cfg5", "qrdm"), ("cfg2_qrp", "qrp")):
        if name == "cfg2_qrp":
            A = inputs.device_cfg("cfg2", seed=1)
        else:
            A = inputs.device_cfg(name, seed=4)
        m, n = A.shape
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
        # scalar-pivot columns: the reference's rank-1 flops (rrqr.py:231), and the one
        # read of the trailing block per column the blocked engine cannot avoid
        f_sc = sum(4.0 * (m - s.n_s) * (n - s.n_s - 1) for s in scal)
        b_sc = sum(8.0 * (m - s.n_s) * (n - s.n_s - 1) for s in scal)
        t_roof = (f_dm + f_sc) / (peak_tf * 1e12) * 1e3          # all of it at the FP64 peak
        t_phased = (f_dm / (peak_tf * 1e12) + b_sc / 6542.4e9) * 1e3  # scalar-pivot phase at HBM speed
        out[name] = {"algo": "qrp" if algo == "qrp" else "qrdm2",
                     "m": m, "n": n, "ms": best, "rank": int(f.info.rank), "outer_steps": len(steps),
                     "scalar_pivot_steps": sum(1 for s in steps if s.fell_back_to_scalar),
                     "gflops_nominal": nominal(m, n) / (best / 1e3) / 1e9 if m >= n else None,
                     "gflops_executed": partial_nominal(m, n, nf) / (best / 1e3) / 1e9 if m >= n else None,
                     "t_roof_ms": t_roof, "roofline_frac": t_roof / best,
                     "t_roof_phased_ms": t_phased, "roofline_phased_frac": t_phased / best,
                     "roofline_note": "t_roof: trailing-update flops (scalar-pivot rank-1 flops counted as "
                                      "BLAS3) at the measured DGEMM peak; phased: the DM steps' flops at the "
                                      "peak plus one HBM read of the trailing block per scalar-pivot column"}
        del work, b0, f
        torch.cuda.empty_cache()
    # cfg3: the batch of 1024 independent 256 x 256 matrices (bench.py --config cfg3 times it alone)
    from paper_2106_03138_b200.batch import factorize_batch, to_batch_work

    w0 = to_batch_work(inputs.cfg3(seed=3, batch=1024), dev)
    wb = w0[0].clone()
    best = 1e30
    for _ in range(3):
        wb.copy_(w0[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        factorize_batch(None, lanes=4, work=(wb, w0[1], w0[2], w0[3]))
        e1.record()
        torch.cuda.synchronize(dev)
        best = min(best, e0.elapsed_time(e1))
    out["cfg3"] = {"algo": "qrdm2", "batch": 1024, "m": 256, "n": 256, "ms": best,
                   "matrices_per_s": 1024 / (best / 1e3), "gflops_nominal": 1024 * nominal(256, 256) / (best / 1e3) / 1e9}
    del w0, wb
    torch.cuda.empty_cache()
    return out


def run_b200(args, rank, world):
    import torch
    import torch.distributed as dist

    from paper_2106_03138_b200 import _lib, inputs, rrqr

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n = args.size
    A = inputs.cfg2(seed=args.seed + rank, n=n)
    params, stop = rrqr.DMParams(), rrqr.StopCriterion()
    lib = _lib.load()

    work0 = rrqr.to_work(A, dev)
    buf0 = work0[0]
    buf = buf0.clone()
    work = (buf, work0[1], work0[2], work0[3])

    def step():
        buf.copy_(buf0)
        return rrqr.factorize(None, params, stop, break_check=True, work=work)

    for _ in range(args.warmup):
        f = step()
    torch.cuda.synchronize(dev)
    last = rrqr.to_result(f)
    steps_log = last.step_log

    peak_tf = fp64_peak_tflops(torch, dev)
    if world > 1:
        dist.barrier()
    lib.dmqr_stats_enable(1)
    _lib.stats(reset=True)
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        ev0.record()
        for _ in range(args.steps):
            f = step()
        ev1.record()
        torch.cuda.synchronize(dev)
    lib.dmqr_stats_enable(0)
    st = _lib.stats(reset=True)
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    ms_step = ms / args.steps
    value = world * nominal(n, n) / (ms_step / 1e3) / 1e9

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
    kmax = min(n, n)
    h2d = 8 * n * n
    d2h = 8 * n * n + 8 * kmax + 8 * n + 16 * len(res.perm.swaps) + 56 * len(res.step_log)
    e2e_val = world * nominal(n, n) / (e2e_step / 1e3) / 1e9
    if world > 1:
        t = torch.tensor([e2e_step], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_val = world * nominal(n, n) / (float(t.item()) / 1e3) / 1e9

    # ---- roofline of the dominant throughput kernels: the DMMA trailing update ----
    # In the default (look-ahead) schedule the trailing GEMM tiles run inside
    # k_spare beside the panel, so their time is hidden; one extra, untimed
    # factorization in the serial schedule times the same tile code
    # (k_trail_a = the G/Z loop, k_trail_b = the C -= Y Wt tiles) alone.
    ftr = trailing_flops(n, n, steps_log)
    os.environ["DMQR_NO_LOOKAHEAD"] = "1"
    try:
        lib.dmqr_stats_enable(1)
        _lib.stats(reset=True)
        step()
        torch.cuda.synchronize(dev)
        st_serial = _lib.stats(reset=True)
        lib.dmqr_stats_enable(0)
    finally:
        del os.environ["DMQR_NO_LOOKAHEAD"]
    tr_ms = st_serial["ms_trailing"]
    achieved = ftr / (tr_ms / 1e3) / 1e12 if tr_ms > 0 else None
    bp = panel_bytes(n, n, steps_log)
    t_roof_ms = max(ftr / (peak_tf * 1e12), bp / (6542.4e9)) * 1e3
    traffic = None
    prof = ROOT / "profiles" / "r01_trailing_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("traffic_bytes_per_launch")
        except Exception:
            traffic = None

    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu:
        from threadpoolctl import threadpool_info

        from oracle import qrdm_oracle as O  # the checker/baseline only

        t0 = time.perf_counter()
        ref = O.qrdm2(A)
        t_cpu = time.perf_counter() - t0
        threads = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
        same = bool(np.array_equal(ref.forward, last.perm.forward)) and ref.rank == last.rank
        cpu = {"value": nominal(n, n) / t_cpu / 1e9, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"one full qrdm2 of the same cfg2 {n}x{n} matrix ({t_cpu:.1f} s) with the numpy "
                         f"oracle port (oracle/qrdm_oracle.py), {threads} BLAS threads of "
                         f"{len(os.sched_getaffinity(0))} host cores; GPU perm/rank identical: {same}"}
    extra = None
    if world == 1 and not args.no_extra:
        extra = other_configs(torch, dev, peak_tf)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg2 qrdm2 {n}x{n} N(0,1) seed {args.seed}+rank", "algo": "qrdm2",
                   "m": n, "n": n, "tau": 0.15, "delta": 0.9, "k_dm": 64, "stop": "eps*n",
                   "rank": last.rank, "outer_steps": len(steps_log),
                   "l2": "matrix (134 MB) + pristine copy exceed the 126 MB L2; each step re-copies the input"},
        "gpu_launches": int(st["kernel_launches"]),
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e2e_step, "path": "paper_2106_03138_b200.qrdm2(pinned host tensor) -> numpy result"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": (achieved / peak_tf) if achieved else None, "traffic": traffic,
                     "kernel": "trailing update tiles (k_trail_a: Y^T C split-K + T^T, k_trail_b: C -= Y Wt; DMMA "
                               "m8n8k4 f64), timed alone in one serial-schedule factorization; the default "
                               "schedule runs the same tiles in k_spare beside the panel",
                     "ms_per_factorization": tr_ms,
                     "peak_source": "cuBLAS DGEMM 8192^3 best-of-5 measured in this run (FP64 peak; "
                                    "MEASURED_PEAKS.json has bf16 only)",
                     "algorithmic_flops_per_step": ftr},
        "step_roofline": {"t_roof_ms": t_roof_ms, "t_step_ms": ms_step, "frac": t_roof_ms / ms_step,
                          "panel_bytes": bp, "hbm_gbs": 6542.4},
        "phases_ms_per_step": {k: st[k] / max(args.steps, 1) for k in
                               ("ms_select", "ms_panel", "ms_trailing", "ms_norms")},
        "phases_note": "look-ahead schedule: ms_panel includes k_spare (previous step's C -= Y Wt and "
                       "G = Q1^T C) running beside the panel; ms_trailing is k_trail_w",
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "other_configs": extra,
    }
    print(json.dumps(line), flush=True)


def run_b200_cfg3(args, rank, world):
    """cfg3: a batch of 1024 independent 256 x 256 matrices sharded over the ranks;
    value = matrices/s of the whole job (NCCL gathers only the small per-matrix outputs)."""
    import torch
    import torch.distributed as dist

    from paper_2106_03138_b200 import _lib, inputs
    from paper_2106_03138_b200.batch import factorize_batch, gather_summaries, shard, summary_tensor, to_batch_work

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    batch = args.batch
    B = inputs.cfg3(seed=3, batch=batch)
    lo, hi = shard(batch, rank, world)
    work0 = to_batch_work(B[lo:hi], dev)
    buf = work0[0].clone()
    work = (buf, work0[1], work0[2], work0[3])

    def step():
        buf.copy_(work0[0])
        return factorize_batch(None, lanes=args.lanes, work=work)

    for _ in range(args.warmup):
        f = step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    _lib.stats(reset=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
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
        full = gather_summaries(summary_tensor(f, dev), batch)
        ranks_all = full[:, 0].cpu().numpy()
    else:
        ranks_all = f.ranks
    ms_step = ms / args.steps
    flops = batch * nominal(256, 256)
    value = batch / (ms_step / 1e3)
    if rank != 0:
        return
    line = {
        "metric": "QRDM matrices/s (cfg3 batch)", "value": value, "unit": "matrices/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg3 qrdm2 batch {batch} x 256x256 (B C + 1e-10 E), sharded over {world} GPU(s)",
                   "lanes": args.lanes, "gflops": flops / (ms_step / 1e3) / 1e9,
                   "rank_histogram": {int(k): int(v) for k, v in zip(*np.unique(ranks_all, return_counts=True))}},
        "gpu_launches": int(st["kernel_launches"]), "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the cfg4 / cfg5 / qrp information block")
    ap.add_argument("--config", default="cfg2", choices=["cfg2", "cfg3"])
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--lanes", type=int, default=4)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if args.impl == "b200":
            import torch
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
            dist.init_process_group("nccl")
        else:
            dist.init_process_group("gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.config == "cfg3":
        run_b200_cfg3(args, rank, world)
    else:
        run_b200(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
