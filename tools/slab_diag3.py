import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2405_19991_b200 as otm
from paper_2405_19991_b200.slab import CudaSlabBackend, LocalComm, SlabDesignRun, SlabSolver
name = "c4"
dims = bench.CONFIGS[name]["dims"]
seed = otm.init_density(dims, otm.InitPattern("iwp", 0.5, seed=0)).rho
B = CudaSlabBackend(3 * (dims[0] + 2) * dims[1] * dims[2])
orig_cap = SlabSolver._capture
def cap(self, fn):
    t0 = time.perf_counter()
    orig_cap(self, fn)
    print("capture", round(time.perf_counter() - t0, 3), "failed", getattr(self, "_graph_failed", False), flush=True)
SlabSolver._capture = cap
orig_solve = SlabSolver.solve
def solve(self, *a, **k):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = orig_solve(self, *a, **k)
    torch.cuda.synchronize(); print("  solve", r, round((time.perf_counter() - t0) * 1e3, 1), "ms", flush=True)
    return r
SlabSolver.solve = solve
comm = LocalComm(1)
for rep in range(2):
    run = SlabDesignRun(bench.make_config(otm, name, 3, 0.0), comm, B, [torch.from_numpy(seed).cuda()])
    while not run.finished:
        torch.cuda.synchronize(); t0 = time.perf_counter()
        run.step()
        torch.cuda.synchronize(); print("iteration", round((time.perf_counter() - t0) * 1e3, 1), flush=True)
