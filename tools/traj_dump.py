"""Run the golden trajectory configs on the device and dump per-iteration g, V,
V*, tensor and V-cycle counts (for comparing against the reference runs in
tests/golden/traj_*.npz).  Usage: python tools/traj_dump.py [names...] [--tol T]"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_19991_b200 as otm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("names", nargs="*", default=["traj_c1_conv", "traj_c2_30", "traj_c3_10", "traj_flat100"])
ap.add_argument("--tol", type=float, default=None)
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out"))
args = ap.parse_args()
os.makedirs(args.out, exist_ok=True)
for name in args.names:
    g = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
    dims = tuple(int(d) for d in g["dims"])
    extra = {} if args.tol is None else {"solver_tol": args.tol}
    cfg = otm.RunConfig(dims=dims, target=otm.ObjectiveSpec("mse", otm.ConductivityTensor(np.asarray(g["target"], float))),
                        filter=otm.FilterSpec(float(g["filter_radius"])),
                        init=otm.InitPattern("iwp", float(g["vf"]), seed=0), max_iter=int(g["max_iter"]), **extra)
    kap = []
    t0 = time.perf_counter()
    try:
        res = otm.run_optimization(cfg, callback=lambda it, fld, r, gv: kap.append(np.array(r.tensor.vec)))
        log, conv, err = res.log, res.converged, ""
    except otm.OptimizationAborted as e:
        log, conv, err = e.partial.log, False, str(e)
    wall = time.perf_counter() - t0
    tag = "" if args.tol is None else f"_tol{args.tol:.0e}"
    np.savez(os.path.join(args.out, f"gpu_{name}{tag}.npz"), g=np.array([r.g for r in log]),
             volfrac=np.array([r.volfrac for r in log]), vstar=np.array([r.vstar for r in log]),
             vcycles=np.array([r.vcycles for r in log]), kappa=np.array(kap), converged=conv, wall_s=wall)
    n = min(len(log), len(g["g"]))
    relg = np.abs(np.array([r.g for r in log[:n]]) - g["g"][:n]) / np.abs(g["g"][:n])
    first = int(np.argmax(relg > 1e-3)) if (relg > 1e-3).any() else -1
    print(f"{name}{tag}: {len(log)} its (ref {len(g['g'])}), converged {conv}, wall {wall:.2f}s, "
          f"max rel g {relg.max():.2e}, first >1e-3 at {first} {err}", flush=True)
