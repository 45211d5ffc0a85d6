"""Break down the end-to-end (public API) time of one c3 structure on the GPU:
context creation, first iteration (graph capture/instantiate), steady iterations."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import bench
import paper_2405_19991_b200 as otm
from paper_2405_19991_b200.optimize import DesignRun

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 500
dims = bench.CONFIGS["c3"]["dims"]
seed = otm.init_density(dims, otm.InitPattern("iwp", 0.5, seed=0)).rho


def now():
    torch.cuda.synchronize()
    return time.perf_counter()


t0 = now()
h = otm.GridHierarchy(dims)
t1 = now()
print(f"GridHierarchy create: {(t1 - t0) * 1e3:.1f} ms", flush=True)
for rep in range(3):
    cfg = bench.make_config(otm, "c3", iters, 0.0, init_field=seed)
    t0 = now()
    run = DesignRun(cfg, hier=h)
    t1 = now()
    run.step()
    t2 = now()
    while not run.finished:
        run.step()
    t3 = now()
    rho = run.rho.cpu().numpy()
    t4 = now()
    print(f"rep {rep}: init {(t1 - t0) * 1e3:.1f} ms, first step {(t2 - t1) * 1e3:.1f} ms, "
          f"rest {(t3 - t2) * 1e3:.1f} ms ({len(run.log)} it), d2h {(t4 - t3) * 1e3:.1f} ms", flush=True)
for rep in range(2):
    cfg = bench.make_config(otm, "c3", iters, 0.0, init_field=seed)
    t0 = now()
    res = otm.run_optimization(cfg)
    t1 = now()
    print(f"run_optimization: {(t1 - t0) * 1e3:.1f} ms ({res.iterations} it)", flush=True)
