"""Several independent c3 structures on one GPU at once (one hierarchy, stream and
host thread each): wall time per structure against one at a time.

    python tools/multi_structure.py [K] [ITERS]

Every hierarchy captures its iteration graph in a sequential warm-up run first
(the launchers' static tensor-map caches are not thread-safe while capturing);
the timed runs only launch captured graphs.
"""
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2405_19991_b200 as otm  # noqa: E402
from paper_2405_19991_b200.optimize import DesignRun  # noqa: E402
from paper_2405_19991_b200.solver import GridHierarchy  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 2
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 500
dims = bench.CONFIGS["c3"]["dims"]
seed = otm.init_density(dims, otm.InitPattern("iwp", bench.CONFIGS["c3"]["vf"], seed=0)).rho
cfg = bench.make_config(otm, "c3", iters, 0.0, init_field=seed)
hiers = [GridHierarchy(dims, material=cfg.material, filter_radius=cfg.filter.radius) for _ in range(K)]


def one(h, out, i):
    run = DesignRun(cfg, hier=h)
    run.run()
    out[i] = run


for h in hiers:                    # capture sequentially
    one(h, [None], 0)
torch.cuda.synchronize()

t0 = time.perf_counter()
for h in hiers:
    one(h, [None], 0)
torch.cuda.synchronize()
seq = time.perf_counter() - t0

outs = [None] * K
threads = [threading.Thread(target=one, args=(h, outs, i)) for i, h in enumerate(hiers)]
t0 = time.perf_counter()
for t in threads:
    t.start()
for t in threads:
    t.join()
torch.cuda.synchronize()
conc = time.perf_counter() - t0
g = [r.log[-1].g for r in outs]
print(f"K={K}: sequential {seq:.3f} s ({seq / K:.3f} s/structure), concurrent {conc:.3f} s "
      f"({conc / K:.3f} s/structure, x{seq / conc:.2f}); final g {np.round(g, 8)}")
