#!/usr/bin/env python
"""Summarise ncu outputs for profiles/ (run in the build container).

  python profiles/summarize.py launches gpurun_out/launches_c3.csv > profiles/r01_launches_c3.md
  python profiles/summarize.py full gpurun_out/prof_c3.ncu-rep > profiles/r01_full_c3.md
"""

import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__waves_per_multiprocessor", "waves"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    gi = h.index("Grid Size") if "Grid Size" in h else None
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("otm::", "")
        if gi is not None and len(sys.argv) > 3 and sys.argv[3] == "grid":
            name += " " + r[gi]
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    print(f"# ncu launch list: {path}\n")
    print("Per-launch device time (`gpu__time_duration.sum`, `--clock-control none`; cold-cache and "
          "serialised by ncu, so compare shares, not absolutes).\n")
    print("| kernel | launches | total µs | avg µs | share |")
    print("|---|---:|---:|---:|---:|")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {c} | {v / 1e3:.1f} | {v / c / 1e3:.2f} | {100 * v / tot:.1f}% |")
    print(f"\nTotal: {tot / 1e3:.1f} µs over {sum(c for c, _ in agg.values())} launches.")


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    print(f"# ncu --set full: {path}\n")
    cols = [m for m, _ in METRICS if m in h]
    print("| kernel | grid | block | " + " | ".join(dict(METRICS)[m] for m in cols) + " |")
    print("|---|---|---|" + "---:|" * len(cols))
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("otm::", "")
        vals = []
        for m in cols:
            u = units[h.index(m)]
            vals.append(f"{r[h.index(m)]} {u}".strip())
        print(f"| `{name}` | {r[h.index('Grid Size')]} | {r[h.index('Block Size')]} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
