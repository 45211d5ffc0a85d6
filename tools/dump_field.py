"""Run the design loop on the GPU and dump the density at given iterations (solver studies).

    python tools/dump_field.py N ITERS [c2|c3]

Writes gpurun_out/fields_N.npz: rho_<it> (float32 filtered densities), vcycles per iteration,
and for every dumped design the residual history of a cold solve to 1e-10
(the asymptotic contraction of the V-cycle-preconditioned CG on that design).
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2405_19991_b200 as otm  # noqa: E402
from paper_2405_19991_b200.optimize import DesignRun  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
stops = [int(s) for s in (sys.argv[2] if len(sys.argv) > 2 else "50,150,300").split(",")]
which = sys.argv[3] if len(sys.argv) > 3 else "c3"
tgt = [0.3, 0.2, 0.1, 0.1, 0.05, 0.05] if which == "c3" else [0.3, 0.2, 0.1, 0, 0, 0]
cfg = otm.RunConfig(dims=(n, n, n), target=otm.ObjectiveSpec("mse", otm.ConductivityTensor(tgt)),
                    init=otm.InitPattern("iwp", 0.5), max_iter=max(stops) + 1, conv_threshold=0.0)
run = DesignRun(cfg)
out, vc = {}, []
while not run.finished:
    rc, rec = run.evaluate()
    vc.append(rec.vcycles)
    if rec.iter in stops:
        out[f"rho_{rec.iter}"] = run.rho_f.cpu().numpy().astype(np.float32)   # filtered density
        print(rec.iter, rec.g, rec.volfrac, flush=True)
    if not run.finished:
        run.update()
out["vcycles"] = np.array(vc)
mp = otm.MaterialParams()
for it in stops:
    rho = out[f"rho_{it}"].astype(np.float64)
    h = otm.GridHierarchy((n, n, n))
    h.build_density(rho, mp)
    h.solve3(None, tol=1e-10, max_vcycles=400)
    hist = np.array(h.residual_history)
    out[f"hist_{it}"] = hist
    k = len(hist)
    rate = (hist[-1] / hist[0]) ** (1.0 / max(k - 1, 1)) if k > 1 else 0.0
    print(f"iter {it}: cold solve to 1e-10: {k} V-cycles, mean contraction {rate:.3f}", flush=True)
np.savez_compressed(f"gpurun_out/fields_{n}_{which}.npz", **out)
