"""Per-launch summary of an ncu report: time, DRAM bytes, achieved GB/s, SM and
DMMA-pipe utilisation.  python tools/ncu_summary.py report.ncu-rep [algorithmic_bytes_expr...]"""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_dmma.avg.pct_of_peak_sustained_active", "launch__grid_size"]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
col = {k: i for i, k in enumerate(h)}


def val(r, k):
    if k not in col or r[col[k]] in ("", "n/a"):
        return float("nan")
    v = float(r[col[k]].replace(",", ""))
    u = units[col[k]]
    return v * {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)


print("| kernel | grid | us | DRAM rd MB | DRAM wr MB | DRAM GB/s | SM thr % | DMMA pipe % |")
print("|---|---:|---:|---:|---:|---:|---:|---:|")
for r in rows[2:]:
    name = r[col["Kernel Name"]].split("(")[0]
    t = val(r, "gpu__time_duration.sum")
    rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
    print(f"| {name} | {r[col['launch__grid_size']]} | {t:.1f} | {rd / 1e6:.2f} | {wr / 1e6:.2f} | "
          f"{(rd + wr) / t / 1e3:.0f} | {val(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
          f"{val(r, 'sm__inst_executed_pipe_dmma.avg.pct_of_peak_sustained_active'):.1f} |")
