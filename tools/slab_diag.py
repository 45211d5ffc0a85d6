"""Slab solver diagnostics: V-cycles and time of one solve at c4 under solver knobs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2405_19991_b200 as otm
from paper_2405_19991_b200.slab import CudaSlabBackend, LocalComm, SlabSolver
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
dims = (n, n, n)
rho = otm.init_density(dims, otm.InitPattern("iwp", 0.5, seed=0)).rho
fld = otm.DensityField(dims, rho, np.zeros(dims))
rf = otm.filter_forward(fld, otm.FilterSpec(1.5))
kap = torch.from_numpy(otm.simp_conductivity(rf, otm.MaterialParams())).cuda()
B = CudaSlabBackend(3 * (n + 2) * n * n)
for knobs in (dict(omega=1.0, omega_coarse=1.0, tolf=0.5), dict(), dict(omega_coarse=0.95)):
    for graph in ("1", "0"):
        os.environ["OTM_SLAB_GRAPH"] = graph
        sv = SlabSolver(dims, LocalComm(1), B, **knobs)
        sv.build_kappa([kap])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cyc = sv.solve(tol=1e-6)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        sv.warm = False
        cyc2 = sv.solve(tol=1e-6)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(knobs, "graph", graph, "cycles", cyc, cyc2, "s", round(t1 - t0, 4), round(t2 - t1, 4), flush=True)
h = otm.GridHierarchy(dims)
h.build(kap)
torch.cuda.synchronize(); t0 = time.perf_counter()
T, c, _ = h.solve3(None, tol=1e-6)
torch.cuda.synchronize(); print("single", c, round(time.perf_counter() - t0, 4))
