"""Summarise an ncu launch list (gpu__time_duration.sum per launch) per kernel,
over the last complete factorization in the list (k_init .. k_finalize).

  python tools/launch_summary.py gpurun_out/launches.csv > profiles/r01_launches_summary.md
"""

import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name).replace("dmqr::", "")
    return name


def main(path):
    hdr, rows = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                rows.append((short(d["Kernel Name"]), float(d["Metric Value"]), d["Grid Size"], d["Block Size"]))
    inits = [i for i, r in enumerate(rows) if r[0] == "k_init"]
    fins = [i for i, r in enumerate(rows) if r[0] == "k_finalize"]
    lo = hi = None
    for a in reversed(inits):
        later = [f for f in fins if f > a]
        if later:
            lo, hi = a, later[0]
            break
    if lo is None:
        print("no complete factorization in the list")
        return
    seg = rows[lo:hi + 1]
    tot = sum(r[1] for r in seg)
    agg = collections.defaultdict(lambda: [0, 0.0, set()])
    for k, t, g, b in seg:
        a = agg[k]
        a[0] += 1
        a[1] += t
        a[2].add(f"{g}x{b}")
    print(f"# ncu launch list: one factorization (launches {lo}..{hi} of {len(rows)})\n")
    print(f"source: `{path}` (`ncu --metrics gpu__time_duration.sum --clock-control none`), "
          f"cold-cache serialised launches; total kernel time {tot / 1e6:.2f} ms over {len(seg)} launches\n")
    print("| kernel | launches | total ms | share | mean us | grid x block |")
    print("|---|---:|---:|---:|---:|---|")
    for k, (c, t, gs) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {c} | {t / 1e6:.3f} | {100 * t / tot:.1f}% | {t / c / 1e3:.1f} | {', '.join(sorted(gs))[:60]} |")


if __name__ == "__main__":
    main(sys.argv[1])
