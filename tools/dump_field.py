"""Run the design loop on the GPU and dump the density at given iterations (solver studies)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2405_19991_b200 as otm  # noqa: E402
from paper_2405_19991_b200.optimize import DesignRun  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
stops = [int(s) for s in (sys.argv[2] if len(sys.argv) > 2 else "50,150,300").split(",")]
cfg = otm.RunConfig(dims=(n, n, n), target=otm.ObjectiveSpec("mse", otm.ConductivityTensor(
    [0.3, 0.2, 0.1, 0.1, 0.05, 0.05])), init=otm.InitPattern("iwp", 0.5), max_iter=max(stops) + 1,
    conv_threshold=0.0)
run = DesignRun(cfg)
out = {}
while not run.finished:
    rc, rec = run.evaluate()
    if rec.iter in stops:
        out[f"rho_{rec.iter}"] = run.rho.cpu().numpy().astype(np.float32)
        print(rec.iter, rec.g, rec.volfrac, flush=True)
    if not run.finished:
        run.update()
np.savez_compressed(f"gpurun_out/fields_{n}.npz", **out)
