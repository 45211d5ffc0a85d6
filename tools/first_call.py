"""Where does the first run_optimization call of a process spend its time?
(cProfile of the first and second c3 calls; not product code.)

    python tools/first_call.py [CONFIG]
"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_19991_b200 as otm  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
dims = bench.CONFIGS[name]["dims"]
t0 = time.perf_counter()
torch.zeros(1, device="cuda")
print(f"cuda init {time.perf_counter() - t0:.3f} s")
seed = otm.init_density(dims, otm.InitPattern("iwp", bench.CONFIGS[name]["vf"], seed=0)).rho
for k in range(4):
    cfg = bench.make_config(otm, name, 500, 0.0, init_field=seed)
    pr = cProfile.Profile()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pr.enable()
    res = otm.run_optimization(cfg)
    torch.cuda.synchronize()
    pr.disable()
    print(f"call {k}: {time.perf_counter() - t0:.4f} s", flush=True)
    if k in (0, 1):
        pstats.Stats(pr).sort_stats("tottime").print_stats(12)
