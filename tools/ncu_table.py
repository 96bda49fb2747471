"""Kernel table from `ncu --set full` reports (raw page):

  python tools/ncu_table.py gpurun_out/prof_cfg2.ncu-rep [more.ncu-rep ...]
"""
import csv
import io
import re
import subprocess
import sys

COLS = [
    ("us", "gpu__time_duration.sum", 1e-3),
    ("DRAM rd MB", "dram__bytes_read.sum", 1e-6),
    ("DRAM wr MB", "dram__bytes_write.sum", 1e-6),
    ("DRAM GB/s", "dram__bytes.sum.per_second", 1e-9),
    ("SM thr %", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("DMMA pipe %", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", 1),
    ("FP64 pipe %", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
    ("grid", "launch__grid_size", 1),
    ("regs", "launch__registers_per_thread", 1),
]


def to_float(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return float("nan")


def unit_scale(unit, name):
    """to base units (ns, bytes, bytes/s)"""
    u = (unit or "").strip()
    if name.endswith("gpu__time_duration.sum"):
        return {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(u, 1.0)
    if "per_second" in name:
        return {"byte/s": 1.0, "Kbyte/s": 1e3, "Mbyte/s": 1e6, "Gbyte/s": 1e9, "Tbyte/s": 1e12}.get(u, 1.0)
    if "bytes" in name:
        return {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
    return 1.0


def main(paths):
    print("| kernel | " + " | ".join(c[0] for c in COLS) + " |")
    print("|---|" + "---:|" * len(COLS))
    for path in paths:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            name = re.sub(r"\(.*", "", d.get("Kernel Name", "?")).replace("void ", "").replace("dmqr::", "")
            vals = []
            for _, key, sc in COLS:
                v = to_float(d.get(key, "nan")) * unit_scale(u.get(key), key) * sc
                vals.append(f"{v:.1f}" if v == v else "-")
            print(f"| {name} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1:])
