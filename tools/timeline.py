"""Per-step panel vs k_spare timing from globaltimer stamps (DMQR_TIMELINE=1)."""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["DMQR_TIMELINE"] = "1"
import numpy as np  # noqa: E402

from paper_2106_03138_b200 import _lib, inputs, rrqr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
A = inputs.cfg2(seed=1, n=n)
work = rrqr.to_work(A)
buf0 = work[0].clone()
for _ in range(2):
    work[0].copy_(buf0)
    f = rrqr.factorize(None, work=work)
out = np.zeros(64 * 16, dtype=np.int64)
_lib.load().dmqr_debug_panel_clocks(f.workspace.data_ptr(), n, n, out.ctypes.data_as(C.c_void_p))
t = out.reshape(-1, 4)[: int(f.info.n_steps)]
print("step  panel_us  spare_start_us  spare_end_us  (relative to the panel start)")
for i, (p0, p1, s0, s1) in enumerate(t):
    if p0 == 0:
        continue
    print(f"{i:4d} {(p1 - p0) / 1e3:9.1f} {(s0 - p0) / 1e3:14.1f} {(s1 - p0) / 1e3:13.1f}")
g = out[512:512 + 8 * 64].reshape(64, 8)[: int(f.info.n_steps)]
print("gram_finish (us from CTA entry): last-CTA start, loaded, Theta start, filter start, plan start, end, masks done, greedy done")
for i, r in enumerate(g[:12]):
    if r[0] == 0:
        continue
    print(i, [round(float(x - r[0]) / 1e3, 1) if x else None for x in r[1:8]])

# ---- kernel spans (dmqr_debug_timeline): start after the dependency wait, end at the last CTA exit
names = ["select", "gram", "gfinish", "swap", "panel", "spare", "ygemm", "trail_w", "trail_a", "guard", "step_end"]
tl = np.zeros(64 * 32 + 1024, dtype=np.int64)  # (the last 1024: k_spare per-CTA debug)
_lib.load().dmqr_debug_timeline(f.workspace.data_ptr(), int(A.shape[0]), int(A.shape[1]), tl.ctypes.data_as(C.c_void_p))
tl = tl[:2048].reshape(64, 32)
ns = int(f.info.n_steps)
U64MAX = np.int64(-1)
rows = []
for s in range(min(ns, 64)):
    r = tl[s]
    t0 = r[0]
    if t0 in (0, U64MAX):
        continue
    spans = {}
    for k, nm in enumerate(names):
        a, b = r[2 * k], r[2 * k + 1]
        if a == U64MAX or b == 0:
            continue
        spans[nm] = ((a - t0) / 1e3, (b - t0) / 1e3)
    nxt = tl[s + 1][0] if s + 1 < 64 and tl[s + 1][0] not in (0, U64MAX) else None
    rows.append((s, spans, (nxt - t0) / 1e3 if nxt is not None else None))
print("\nstep: kernel [start, end] us from the step's k_select start; 'next' = next step's k_select start")
for s, spans, nxt in rows[:4] + rows[len(rows) // 2: len(rows) // 2 + 2]:
    print(s, " ".join(f"{k}[{a:.1f},{b:.1f}]" for k, (a, b) in spans.items()), f"next {nxt}")
mid = [r for r in rows if 4 <= r[0] < len(rows) - 8]
if mid:
    print("\nmean over steps 4..%d (us): start / end / dur" % (len(rows) - 9))
    for nm in names:
        v = [r[1][nm] for r in mid if nm in r[1]]
        if v:
            a = np.mean([x[0] for x in v]); b = np.mean([x[1] for x in v])
            print(f"  {nm:9s} {a:7.1f} {b:7.1f} {b - a:7.1f}  (n={len(v)})")
    print("  step      ", np.mean([r[2] for r in mid if r[2]]))

# k_trail_w's first Wt tile (slots 22..26): staged-issue, landed, R12 done, tile done, close start; relative to the kernel's span start
print("\nk_trail_w CTA 0 (us after the span start): copies issued, landed, R12 stored, tile done, close start, span end")
for s in (8, 20, 32, 33, 48):
    r = tl[s]
    if r[14] in (0, U64MAX):
        continue
    print(s, [round(float(r[k] - r[14]) / 1e3, 1) if r[k] else None for k in (22, 23, 24, 25, 26, 15)])

# k_spare phases (slots 28, 29, 31): Q1 seen, phase 1 (pending update) end, phase 2 (G tiles) end; us after k_spare's start
print("\nk_spare (us after its start): Q1 seen, phase-1 end, phase-2 end, span end; panel end")
for s in (1, 2, 4, 8, 12, 16, 20, 32, 48):
    r = tl[s]
    if r[10] in (0, U64MAX):
        continue
    f = lambda k: round(float(r[k] - r[10]) / 1e3, 1) if r[k] not in (0, U64MAX) else None
    print(s, [f(28), f(29), f(31), f(11)], f(9))
