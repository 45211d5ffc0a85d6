"""Run N design iterations of c3 through DesignRun (for ncu launch lists of the
steady state: skip the first iterations' launches with --launch-skip).

    python tools/profile_run.py ITERS [CONFIG] [graph]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bench
import paper_2405_19991_b200 as otm
from paper_2405_19991_b200.optimize import DesignRun

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40
cfg_name = sys.argv[2] if len(sys.argv) > 2 else "c3"
dims = bench.CONFIGS[cfg_name]["dims"]
seed = otm.init_density(dims, otm.InitPattern("iwp", bench.CONFIGS[cfg_name]["vf"], seed=0)).rho
cfg = bench.make_config(otm, cfg_name, iters, 0.0, init_field=seed)
run = DesignRun(cfg)
import time
torch.cuda.synchronize()
t0 = time.perf_counter()
if len(sys.argv) > 3 and sys.argv[3] == "graph":
    run.run()                                   # device-resident iteration graph
else:
    while not run.finished:
        run.step()
torch.cuda.synchronize()
print(f"wall {time.perf_counter() - t0:.4f} s")
lib = run.hier.ctx.lib
print("launches", lib.otm_launch_count(run.hier.ctx.h), "iterations", len(run.log),
      "vcycles", sum(r.vcycles for r in run.log))
