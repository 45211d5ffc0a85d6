"""Generate golden vectors by running the REAL reference package.

Runs only in the build container, where the read-only reference lives at
/root/reference/pkg/src (importable as ``opentm``).
The outputs (small .npz files next to this script) are committed; neither the
GPU box nor the test-suite needs the reference afterwards.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--big]

``--big`` adds the 64^3 / 128^3 first-iteration fixtures (~2 min of CPU).
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import opentm  # noqa: F401
    return opentm


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}: {sorted(arrays)}")


def gen_element(ot):
    t = ot.build_templates()
    save("element.npz", K0=t.K0, f0=t.f0)


def gen_filter(ot):
    rng = np.random.default_rng(100)
    rho = rng.uniform(0, 1, (6, 7, 8))
    g = rng.standard_normal((6, 7, 8))
    out = {"rho": rho, "g": g}
    for r in (1.5, 2.0):
        spec = ot.FilterSpec(r)
        fld = ot.DensityField(rho.shape, rho, np.zeros(rho.shape))
        offs, w = spec.offsets_and_weights()
        tag = str(r).replace(".", "p")
        out[f"fwd_{tag}"] = ot.filter_forward(fld, spec)
        out[f"bwd_{tag}"] = ot.filter_backward(fld, spec, g)
        out[f"offs_{tag}"] = offs
        out[f"w_{tag}"] = w
    sym = rng.uniform(0, 1, (6, 6, 4))
    fld = ot.DensityField(sym.shape, sym.copy(), np.zeros(sym.shape))
    ot.project_central_symmetry(fld)
    out["sym_in"] = sym
    out["sym_out"] = fld.rho
    save("filter.npz", **out)


def gen_operator(ot):
    from opentm.solver import GridHierarchy, apply_K, assemble_macro_load
    rng = np.random.default_rng(101)
    out = {}
    for tag, dims in (("a", (4, 5, 6)), ("b", (6, 6, 6)), ("c", (8, 4, 2)), ("d", (6, 4, 1))):
        kap = rng.uniform(1e-4, 1.0, dims)
        T = rng.standard_normal(dims)
        h = GridHierarchy(dims, dtype="float64")
        h.build(kap)
        out[f"kappa_{tag}"] = kap
        out[f"T_{tag}"] = T
        out[f"KT_{tag}"] = apply_K(h.levels[0], T)
        out[f"f_{tag}"] = np.stack([assemble_macro_load(h, i) for i in range(3)])
    # level chains and child-mean kappa
    h = GridHierarchy((16, 16, 16), dtype="float64")
    kap = rng.uniform(0.1, 1.0, (16, 16, 16))
    h.build(kap)
    out["chain_kappa16"] = kap
    for li, lev in enumerate(h.levels):
        out[f"chain_level{li}_kappa"] = lev.kappa
        out[f"chain_level{li}_template"] = lev.template
    chains = {}
    for dims in ((16, 16, 16), (32, 32, 32), (128, 128, 128), (100, 100, 1), (12, 12, 12), (64, 32, 16)):
        chains[str(dims)] = [lev.dims for lev in GridHierarchy(dims).levels]
    out["chain_dims_keys"] = np.array(list(chains.keys()))
    for i, (k, v) in enumerate(chains.items()):
        out[f"chain_dims_{i}"] = np.array(v)
    save("operator.npz", **out)


def gen_solve(ot):
    from opentm.solver import GridHierarchy, solve_equation
    rng = np.random.default_rng(102)
    kap = rng.uniform(0.05, 1.0, (8, 8, 8))
    f = rng.standard_normal((8, 8, 8))
    f -= f.mean()
    h = GridHierarchy((8, 8, 8), dtype="float64")
    h.build(kap)
    T, cyc = solve_equation(h, f, tol=1e-10)
    hist = np.array(h.residual_history)
    x0 = rng.standard_normal((8, 8, 8))
    T2, cyc2 = solve_equation(h, f, tol=1e-10, x0=x0)
    save("solve.npz", kappa=kap, f=f, T=T, cycles=cyc, history=hist, x0=x0, T_warm=T2,
         cycles_warm=cyc2)


def _homog_fixture(ot, name, rho, target, tol=1e-10):
    mp = ot.MaterialParams()
    spec = ot.FilterSpec(1.5)
    fld = ot.DensityField(rho.shape, rho.copy(), np.zeros(rho.shape))
    rho_f = ot.filter_forward(fld, spec)
    h = ot.GridHierarchy(rho.shape, dtype="float64")
    res = ot.homogenize(h, rho_f, mp, tol=tol)
    obj = ot.ObjectiveSpec("mse", ot.ConductivityTensor(target))
    g, dG = ot.eval_objective(obj, res.tensor)
    sens_f = ot.tensor_sensitivity(res, dG)
    sens = ot.filter_backward(fld, spec, sens_f)
    save(name, rho=rho, rho_f=rho_f, target=np.asarray(target, float), kappa_h=res.tensor.vec,
         g=g, dG=dG, sens_f=sens_f, sens=sens, T=np.stack(res.T_fields),
         pair_energy=res.pair_energy, vcycles=res.vcycles)


def gen_homog(ot):
    rng = np.random.default_rng(103)
    _homog_fixture(ot, "homog_rand8.npz", rng.uniform(0.1, 1.0, (8, 8, 8)),
                   [0.3, 0.2, 0.1, 0.1, 0.05, 0.05])
    iwp = ot.init_density((16, 16, 16), ot.InitPattern("iwp", 0.3, seed=0)).rho
    _homog_fixture(ot, "homog_iwp16.npz", iwp, [0.1, 0.1, 0.1, 0, 0, 0])
    _homog_fixture(ot, "homog_rand_6x8x10.npz", rng.uniform(0.05, 1.0, (6, 8, 10)),
                   [0.3, 0.2, 0.1, 0.0, 0.0, 0.0])


def gen_oc(ot):
    from opentm.optimize import GovernorState, OCParams, governor_update, oc_update
    rng = np.random.default_rng(104)
    out = {}
    cases = []
    for k in range(6):
        rho = rng.uniform(0.0, 1.0, (8, 8, 8)) if k % 2 else rng.uniform(0.1, 0.9, (8, 8, 8))
        sens = rng.standard_normal(rho.shape) * (1e-3 if k < 3 else 1.0)
        if k == 4:
            sens = -np.abs(sens)  # all descent: slack step
        bound = float(rho.mean()) + (-0.02, 0.0, 0.01, -0.005, 0.5, 0.003)[k]
        params = OCParams(step_limit=(0.02, 0.05)[k % 2])
        new, info = oc_update(rho, sens, bound, params)
        out[f"rho_{k}"] = rho
        out[f"sens_{k}"] = sens
        out[f"bound_{k}"] = bound
        out[f"step_{k}"] = params.step_limit
        out[f"new_{k}"] = new
        out[f"lam_{k}"] = info["lam"]
        out[f"active_{k}"] = info["active"]
        cases.append(k)
    out["ncases"] = len(cases)
    # governor trajectory
    st = GovernorState()
    rho = rng.uniform(0.2, 0.9, (4, 4, 4))
    gs = [1e-2, 5e-3, 5e-5, 4e-5, 2e-4, 2e-4, 2.05e-4, 2.1e-4, 2.0e-4, 2.02e-4, 2.01e-4, 5e-5]
    trace = []
    for g in gs:
        v = governor_update(st, g, rho, 3.0)
        trace.append([v, st.df, st.gap, st.count, float(st.reduced), st.current_decrease])
    out["gov_rho"] = rho
    out["gov_g"] = np.array(gs)
    out["gov_trace"] = np.array(trace)
    save("oc.npz", **out)


def gen_trajectory(ot, dims=(32, 32, 32), iters=80, name="traj_c1.npz",
                   target=(0.1, 0.1, 0.1, 0, 0, 0), vf=0.3):
    from opentm.optimize import RunConfig, run_optimization
    obj = ot.ObjectiveSpec("mse", ot.ConductivityTensor(list(target)))
    cfg = RunConfig(dims=dims, target=obj, init=ot.InitPattern("iwp", vf, seed=0), max_iter=iters)
    first = {}

    def cb(it, fld, result, g):
        if it == 1:
            first["kappa_h"] = result.tensor.vec.copy()
            first["rho_f"] = result.rho_filtered.copy()

    t0 = time.perf_counter()
    res = run_optimization(cfg, callback=cb)
    wall = time.perf_counter() - t0
    log = res.log
    save(name, g=np.array([r.g for r in log]), volfrac=np.array([r.volfrac for r in log]),
         volfrac_filtered=np.array([r.volfrac_filtered for r in log]),
         vstar=np.array([r.vstar for r in log]), vcycles=np.array([r.vcycles for r in log]),
         rho_final=res.field.rho, kappa_final=res.kappa.vec, kappa_first=first["kappa_h"],
         converged=res.converged, iterations=res.iterations, wall_s=wall,
         target=np.array(target, float), vf=vf)


def gen_big(ot):
    for tag, dims, target, vf in (("c2", (64, 64, 64), [0.3, 0.2, 0.1, 0, 0, 0], 0.5),
                                  ("c3", (128, 128, 128), [0.3, 0.2, 0.1, 0.1, 0.05, 0.05], 0.5)):
        rho = ot.init_density(dims, ot.InitPattern("iwp", vf, seed=0)).rho
        mp = ot.MaterialParams()
        spec = ot.FilterSpec(1.5)
        fld = ot.DensityField(dims, rho.copy(), np.zeros(dims))
        t0 = time.perf_counter()
        rho_f = ot.filter_forward(fld, spec)
        h = ot.GridHierarchy(dims, dtype="float64")
        res = ot.homogenize(h, rho_f, mp, tol=1e-6)
        obj = ot.ObjectiveSpec("mse", ot.ConductivityTensor(target))
        g, dG = ot.eval_objective(obj, res.tensor)
        sens = ot.filter_backward(fld, spec, ot.tensor_sensitivity(res, dG))
        wall = time.perf_counter() - t0
        rng = np.random.default_rng(7)
        idx = rng.integers(0, rho.size, 4096)
        save(f"first_{tag}.npz", dims=np.array(dims), target=np.array(target, float), vf=vf,
             kappa_h=res.tensor.vec, g=g, dG=dG, sens_idx=idx, sens_sample=sens.ravel()[idx],
             sens_absmax=np.abs(sens).max(), sens_sum=sens.sum(), vcycles=res.vcycles,
             wall_s=wall)


SOLVER_TOL = None   # --tol: the same runs at another solver tolerance (chaos envelope)


def _run_logged(ot, name, dims, target, vf, max_iter, filt=1.5):
    """Full reference run; stores the per-iteration log, the tensor after every
    iteration and per-iteration wall times (the CPU-baseline sample)."""
    from opentm.optimize import RunConfig, run_optimization
    obj = ot.ObjectiveSpec("mse", ot.ConductivityTensor(np.array(target, float)))
    extra = {}
    if SOLVER_TOL is not None:
        extra["solver_tol"] = SOLVER_TOL
        name = name.replace(".npz", f"_tol{SOLVER_TOL:.0e}.npz".replace("-0", "-"))
    cfg = RunConfig(dims=dims, target=obj, filter=ot.FilterSpec(filt),
                    init=ot.InitPattern("iwp", vf, seed=0), max_iter=max_iter, **extra)
    kap, stamps = [], [time.perf_counter()]

    def cb(it, fld, result, g):
        kap.append(result.tensor.vec.copy())
        stamps.append(time.perf_counter())

    t0 = time.perf_counter()
    res = run_optimization(cfg, callback=cb)
    wall = time.perf_counter() - t0
    log = res.log
    rho = res.field.rho
    save(name, dims=np.array(dims), target=np.array(target, float), vf=vf, filter_radius=filt,
         max_iter=max_iter, g=np.array([r.g for r in log]),
         volfrac=np.array([r.volfrac for r in log]),
         volfrac_filtered=np.array([r.volfrac_filtered for r in log]),
         vstar=np.array([r.vstar for r in log]), vcycles=np.array([r.vcycles for r in log]),
         iter_ms=np.array([r.ms for r in log]), kappa=np.array(kap),
         iter_wall_s=np.diff(np.array(stamps)), kappa_final=res.kappa.vec,
         rho_sum=float(rho.sum()), rho_sq=float((rho * rho).sum()),
         rho_final=(rho.astype(np.float32) if rho.size <= 40000 else np.zeros(0)),
         converged=res.converged, iterations=res.iterations, wall_s=wall)


def gen_long(ot, which):
    """Multi-iteration trajectories of the headline configs."""
    if which == "c1conv":   # config 1 to convergence (reference: it 237, g 9.98e-5)
        _run_logged(ot, "traj_c1_conv.npz", (32, 32, 32), [0.1, 0.1, 0.1, 0, 0, 0], 0.3, 500)
    elif which == "c2":     # config 2, 30 iterations
        _run_logged(ot, "traj_c2_30.npz", (64, 64, 64), [0.3, 0.2, 0.1, 0, 0, 0], 0.5, 30)
    elif which == "c3":     # config 3, 3 iterations
        _run_logged(ot, "traj_c3_3.npz", (128, 128, 128), [0.3, 0.2, 0.1, 0.1, 0.05, 0.05], 0.5, 3)
    elif which == "c3x10":  # config 3, 10 iterations
        _run_logged(ot, "traj_c3_10.npz", (128, 128, 128), [0.3, 0.2, 0.1, 0.1, 0.05, 0.05], 0.5, 10)
    elif which == "c4x2":   # config 4 (256^3, the C3 target), 2 iterations: k10 nz = 256, lockstep tiles
        _run_logged(ot, "traj_c4_2.npz", (256, 256, 256), [0.3, 0.2, 0.1, 0.1, 0.05, 0.05], 0.5, 2)
    elif which == "flat":   # tests/test_acceptance.py:144-158 (100x100x1, r = 2, NaN targets)
        _run_logged(ot, "traj_flat100.npz", (100, 100, 1), [0.4, 0.2, np.nan, 0.05, np.nan, np.nan],
                    0.5, 500, filt=2.0)
    else:
        raise ValueError(which)


def gen_io(ot):
    """Reference-rendered bytes of every output file (io.py:125-171) for a synthetic
    result, plus the CLI's gallery target list (cli.py:251-283)."""
    import tempfile
    from opentm.cli import enumerate_gallery_targets
    from opentm.io import write_outputs
    from opentm.optimize import IterationRecord, Model, OCParams, OptimizationResult, RunConfig
    rng = np.random.default_rng(105)
    rho = rng.uniform(0, 1, (5, 4, 3))
    target = np.array([0.3, 0.2, np.nan, 0.05, np.nan, 0.01])
    kap = np.array([0.31, 0.19, 0.11, 0.049, 0.002, 0.0101])
    cfg = RunConfig(dims=(5, 4, 3), target=ot.ObjectiveSpec("rel", ot.ConductivityTensor(target)),
                    material=ot.MaterialParams(1.0, 1e-3, 3.5), filter=ot.FilterSpec(2.0),
                    init=ot.InitPattern("random", 0.4, seed=7), model=Model("fixed"), volume_bound=0.4,
                    oc=OCParams(0.002, 0.03, 0.5), max_iter=9, symmetry="central", solver_tol=1e-7)
    its = np.arange(1, 5)
    gs = rng.uniform(1e-6, 1, 4)
    vols = rng.uniform(0.2, 0.6, 4)
    vst = rng.uniform(0.2, 0.6, 4)
    cyc = np.array([12, 7, 9, 30])
    ms = rng.uniform(0.5, 900.0, 4)
    log = [IterationRecord(int(i), float(g), float(v), float(v) * 0.9, float(s), int(c), float(m))
           for i, g, v, s, c, m in zip(its, gs, vols, vst, cyc, ms)]
    res = OptimizationResult(field=ot.DensityField((5, 4, 3), rho, np.zeros((5, 4, 3))),
                             kappa=ot.ConductivityTensor(kap), log=log, converged=False, iterations=4, config=cfg)
    out = {"rho": rho, "target": target, "kappa": kap, "its": its, "gs": gs, "vols": vols, "vst": vst,
           "cyc": cyc, "ms": ms}
    with tempfile.TemporaryDirectory() as d:
        write_outputs(res, d, vtk=True, manifest_extra={"aborted": True, "config_file": None})
        for name in ("rho.otm", "kappa.txt", "log.csv", "manifest.json", "rho.vti"):
            out["file_" + name.replace(".", "_")] = np.frombuffer(open(os.path.join(d, name), "rb").read(),
                                                                  dtype=np.uint8)
    raw, feas = enumerate_gallery_targets([0.3, 0.2, 0.1], 0.05)
    out["gallery_raw"] = np.array(raw)
    out["gallery_feasible"] = np.array(feas)
    raw2, feas2 = enumerate_gallery_targets([0.5, 0.3, 0.2], 0.04)
    out["gallery2_raw"] = np.array(raw2)
    out["gallery2_feasible"] = np.array(feas2)
    save("io.npz", **out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only", default=None)
    ap.add_argument("--long", default=None, help="c1conv | c2 | c3 | c3x10 | c4x2 | flat")
    ap.add_argument("--tol", type=float, default=None, help="solver_tol of the --long run")
    args = ap.parse_args()
    global SOLVER_TOL
    SOLVER_TOL = args.tol
    ot = _ref()
    if args.long:
        t0 = time.perf_counter()
        gen_long(ot, args.long)
        print(f"  [long {args.long}] {time.perf_counter() - t0:.1f}s")
        return
    steps = {"element": gen_element, "filter": gen_filter, "operator": gen_operator,
             "solve": gen_solve, "homog": gen_homog, "oc": gen_oc, "traj": gen_trajectory, "io": gen_io}
    if args.big:
        steps["big"] = gen_big
    for name, fn in steps.items():
        if args.only and name != args.only:
            continue
        t0 = time.perf_counter()
        fn(ot)
        print(f"  [{name}] {time.perf_counter() - t0:.1f}s")


if __name__ == "__main__":
    main()
