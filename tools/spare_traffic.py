"""profiles/r02_spare_traffic.json from an ncu metrics pass over every k_spare launch of one cfg2
factorization (bench.py reads `traffic_bytes_per_launch` for roofline.traffic):

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__ops_path_tensor_src_fp64.sum \
      --clock-control none -k regex:k_spare --csv --log-file gpurun_out/spare_traffic.csv python tools/ab_time.py 4096 0
  python tools/spare_traffic.py gpurun_out/spare_traffic.csv
"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
iname, imet, iunit, ival, iid = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6, "": 1.0, "inst": 1.0}
tot, ids = {}, set()
for r in rows[1:]:
    if "k_spare" not in r[iname]:
        continue
    ids.add(r[iid])
    v = float(r[ival].replace(",", "")) * scale.get(r[iunit], 1.0)
    tot[r[imet]] = tot.get(r[imet], 0.0) + v
n = len(ids)
rd, wr = tot["dram__bytes_read.sum"], tot["dram__bytes_write.sum"]
# algorithmic bytes of a launch, averaged over the 63 steps of cfg2 4096^2 with a pending update (l = 64):
# phase 1 reads and writes the block below the previous step's R rows (16 m' n'' B), phase 2 reads it again (8 m' n'' B)
m = 4096
alg = sum(24.0 * (m - 64 * s) * (m - 64 * s - 64) for s in range(1, 64)) / 64
out = {
    "kernel": "k_spare<0>",
    "launches": n,
    "traffic_bytes_per_launch": (rd + wr) / n,
    "dram_read_bytes": rd,
    "dram_write_bytes": wr,
    "algorithmic_bytes_per_launch": alg,
    "kernel_ms_serialised": tot["gpu__time_duration.sum"] / 1e6,
    "fp64_tensor_ops": tot.get("sm__ops_path_tensor_src_fp64.sum"),
    "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
              "sm__ops_path_tensor_src_fp64.sum --clock-control none -k regex:k_spare python tools/ab_time.py 4096 0 "
              "(all k_spare launches of one cfg2 factorization, serialised by ncu; tools/spare_traffic.py)",
    "note": "algorithmic bytes per launch: phase 1 reads and writes the trailing block below the previous step's R "
            "rows (16 m' n'' B) and phase 2 reads it again for G = Q1^T C (8 m' n'' B), averaged over the launches "
            "(Y, Q1, Wt are small and L2-resident). Traffic below the algorithmic bytes: the 126 MB L2 keeps part of "
            "the block between the phases and between steps.",
}
(ROOT / "profiles" / "r02_spare_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
