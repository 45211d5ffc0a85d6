"""DRAM traffic per launch of the level-0 stencils and the fp64 defect kernel from an
ncu --set full report, against their algorithmic bytes.

    python tools/traffic.py REPORT.ncu-rep CONFIG NX  > profiles/rNN_traffic_CONFIG.json

Only launches on the finest level (template argument NZ == the grid's nz) count.
Algorithmic bytes per vertex: smooth_res / jacobi 44, spmv 28 (3 fp32 cases), the
fp64 defect 44 (T 24 + kappa 8 + r32 12).
"""
import csv
import io
import json
import re
import statistics
import subprocess
import sys

rep, cfg, nx = sys.argv[1], sys.argv[2], int(sys.argv[3])
n = nx ** 3
ALG = {"k10_smooth_res": 44, "k10_jacobi": 44, "k10_spmv": 28, "k_res64w": 44, "k_res64p": 44, "k_load_means_x": 8,
       "k_tensor_x": 32, "k_sens_x": 40, "k_filter_b<2>": 28, "k_filter_b<1>": 16}
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
per, times = {}, {}
for row in rows[2:]:
    name = row[h.index("Kernel Name")]
    m = re.search(r"(k10_smooth_res|k10_jacobi|k10_spmv|k_res64w|k_res64p)<([^>]*)>", name)
    if m:
        args = [a.strip() for a in m.group(2).split(",")]
        nums = [int(a) for a in args if a.lstrip("-").isdigit()]
        nz = nums[1] if m.group(1) == "k10_jacobi" and len(nums) > 1 else nums[0]
        if nz != nx:
            continue
    else:
        m = re.search(r"(k_tensor_x|k_sens_x|k_load_means_x|k_filter_b<[12]>)", name)
        if not m:
            continue
    num = lambda c: float(row[h.index(c)].replace(",", ""))          # base units (bytes, ns)
    b = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    unit = 1.0
    key = f"{m.group(1)}<{m.group(2)}>" if m.lastindex and m.lastindex >= 2 else m.group(1)
    per.setdefault(key, []).append(b * unit)
    times.setdefault(key, []).append(num("gpu__time_duration.sum") * 1e-3)
out = {"source": f"ncu --set full --clock-control none of the finest-level kernels of {cfg} ({nx}^3), {rep}",
       "per_launch_dram_bytes": {k: statistics.mean(v) for k, v in per.items()},
       "per_launch_algorithmic_bytes": {k: ALG.get(k, ALG.get(k.split("<")[0], 0)) * n for k in per},
       "per_launch_us_ncu": {k: statistics.mean(v) for k, v in times.items()}}
st = [k for k in per if k.startswith("k10")]
if st:
    out["mean_dram_bytes"] = statistics.mean(out["per_launch_dram_bytes"][k] for k in st)
    out["mean_algorithmic_bytes"] = statistics.mean(out["per_launch_algorithmic_bytes"][k] for k in st)
print(json.dumps(out, indent=1))
