"""Host-side share of the design loop: wall time of N c3 iterations vs the time the
host spends waiting for the device (OTM_STATS counters).  python tools/hostgap.py [iters]"""
import os
import sys
import time

os.environ["OTM_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2405_19991_b200 as otm
from paper_2405_19991_b200.optimize import DesignRun

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
dims = bench.CONFIGS["c3"]["dims"]
seed = otm.init_density(dims, otm.InitPattern("iwp", 0.5, seed=0)).rho
hier = otm.GridHierarchy(dims)
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    cfg = bench.make_config(otm, "c3", iters, 0.0, init_field=torch.from_numpy(seed).cuda())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run = DesignRun(cfg, hier=hier)
    while not run.finished:
        run.step()
    torch.cuda.synchronize()
    print(f"rep {rep}: {iters} iterations in {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
