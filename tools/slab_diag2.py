"""Per-iteration V-cycles and time of the slab design loop vs the single-GPU loop (c4, 5 its)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2405_19991_b200 as otm
from paper_2405_19991_b200.slab import CudaSlabBackend, LocalComm, SlabDesignRun
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
dims = bench.CONFIGS[name]["dims"]
seed = otm.init_density(dims, otm.InitPattern("iwp", bench.CONFIGS[name]["vf"], seed=0)).rho
B = CudaSlabBackend(3 * (dims[0] + 2) * dims[1] * dims[2])
for graph in ("1", "0"):
    os.environ["OTM_SLAB_GRAPH"] = graph
    for rep in range(2):
        run = SlabDesignRun(bench.make_config(otm, name, 5, 0.0), LocalComm(1), B, [torch.from_numpy(seed).cuda()])
        ts = []
        while not run.finished:
            torch.cuda.synchronize(); t0 = time.perf_counter()
            run.step()
            torch.cuda.synchronize(); ts.append(round((time.perf_counter() - t0) * 1e3, 1))
        print("graph", graph, "rep", rep, "vcycles", [r.vcycles for r in run.log], "ms", ts, flush=True)
r = otm.run_optimization(bench.make_config(otm, name, 5, 0.0, init_field=seed))
print("single vcycles", [x.vcycles for x in r.log], [round(x.ms, 1) for x in r.log])
