"""Per-leg device time of the slab design loop at N = 1 (in-process slab, c4 = 256^3)
against the single-GPU graph path's iteration phases: where the slab path's extra
time goes.  python tools/slab_legs.py [N] [ITERS]"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_19991_b200 as otm  # noqa: E402
from paper_2405_19991_b200 import _lib  # noqa: E402
from paper_2405_19991_b200.optimize import DesignRun  # noqa: E402
from paper_2405_19991_b200.slab import CudaSlabBackend, LocalComm, SlabDesignRun  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dims = (n, n, n)
seed = otm.init_density(dims, otm.InitPattern("iwp", 0.5, seed=0)).rho
cfg = bench.make_config(otm, "c4", iters, 0.0, init_field=seed)
B = CudaSlabBackend(3 * (n + 2) * n * n)
legs = collections.defaultdict(float)


def timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        legs[name] += time.perf_counter() - t0
        return r
    return w


comm = LocalComm(1)                     # one transport: the second run reuses the cached solver
for rep in range(2):
    legs.clear()
    run = SlabDesignRun(cfg, comm, B, [torch.from_numpy(seed).cuda()])
    run.solver.solve = timed("solve", run.solver.solve)
    run.solver.build_kappa = timed("build", run.solver.build_kappa)
    run.solver.tensor = timed("tensor", run.solver.tensor)
    B.filter = timed("filter", B.filter) if rep == 0 else B.filter
    B.sensitivity = timed("sens", B.sensitivity) if rep == 0 else B.sensitivity
    run.update = timed("oc", run.update)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    while not run.finished:
        run.step()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
print(f"slab N=1 {n}^3, {iters} iterations: {wall * 1e3 / iters:.2f} ms/iteration; legs ms/iteration:",
      {k: round(v * 1e3 / iters, 2) for k, v in legs.items()},
      "vcycles", sum(r.vcycles for r in run.log), flush=True)
# single-GPU graph path, same workload
sd = torch.from_numpy(seed).cuda()
for rep in range(2):
    r = DesignRun(bench.make_config(otm, "c4", iters, 0.0, init_field=sd))
    lib = r.hier.ctx.lib
    lib.otm_stats_reset(r.hier.ctx.h)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r.run()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
import ctypes as C  # noqa: E402
ph = (C.c_double * 4)()
lib.otm_loop_phases(r.hier.ctx.h, ph)
print(f"single {n}^3: {wall * 1e3 / iters:.2f} ms/iteration; phases ms/iteration:",
      [round(x / iters, 2) for x in ph], "vcycles", sum(x.vcycles for x in r.log), flush=True)
print("slab pcg graph:", run.solver._pcg_graph is not None, "failed:", getattr(run.solver, "_graph_failed", None))
