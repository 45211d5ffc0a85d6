"""Launch list of the slab design loop at N = 1 (in-process, c4 = 256^3) for ncu:
ITERS warm iterations, then 2 iterations inside the NVTX range "steady".

    ncu --nvtx --nvtx-include "steady/" --metrics gpu__time_duration.sum \
        --clock-control none --csv python tools/slab_launches.py [N] [ITERS]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_19991_b200 as otm  # noqa: E402
from paper_2405_19991_b200.slab import CudaSlabBackend, LocalComm, SlabDesignRun  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dims = (n, n, n)
seed = otm.init_density(dims, otm.InitPattern("iwp", 0.5, seed=0)).rho
cfg = bench.make_config(otm, "c4", warm + 2, 0.0, init_field=seed)
B = CudaSlabBackend(3 * (n + 2) * n * n)
run = SlabDesignRun(cfg, LocalComm(1), B, [torch.from_numpy(seed).cuda()])
for _ in range(warm):
    run.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("steady")
while not run.finished:
    run.step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("vcycles", [r.vcycles for r in run.log])
