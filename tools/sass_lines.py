"""Aggregate ncu SASS-level stall samples by CUDA source line.

  nvdisasm -g <cubin> > all_g.sass
  ncu -i rep --page source --csv --print-source sass > src.csv
  python tools/sass_lines.py all_g.sass src.csv <mangled kernel name> [top]
"""
import csv
import re
import sys
from collections import defaultdict


def line_map(path, fn):
    m, cur, inside = {}, None, False
    for ln in open(path):
        if ".text." in ln and ":" in ln and fn in ln and ln.strip().startswith(".text"):
            inside = True
            continue
        if inside and ln.startswith(".section") or (inside and ln.strip().startswith(".text.") and fn not in ln):
            if m:
                break
        if not inside:
            continue
        g = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if g:
            cur = (g.group(1).split("/")[-1], int(g.group(2)))
            continue
        a = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if a and cur:
            m[int(a.group(1), 16)] = cur
    return m


def main():
    sass, src, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    amap = line_map(sass, fn)
    rows = list(csv.reader(open(src)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    ia, isamp = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
    agg = defaultdict(int)
    reasons = defaultdict(lambda: defaultdict(int))
    rcols = [(i, k[6:]) for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
    tot = 0
    base = None
    for r in rows[hdr + 1:]:
        if len(r) <= isamp:
            continue
        try:
            addr = int(r[ia], 16)
            s = int(r[isamp] or 0)
        except ValueError:
            continue
        if base is None:
            base = addr
        key = amap.get(addr - base, ("?", 0))
        agg[key] += s
        tot += s
        for i, k in rcols:
            try:
                reasons[key][k] += int(r[i] or 0)
            except ValueError:
                pass
    print("total samples", tot, "mapped lines", len(agg))
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        top3 = sorted(reasons[k].items(), key=lambda kv: -kv[1])[:3]
        print(f"{v:7d} {100 * v / max(tot, 1):5.1f}%  {k[0]}:{k[1]}  " + " ".join(f"{a}={b}" for a, b in top3 if b))


if __name__ == "__main__":
    main()
