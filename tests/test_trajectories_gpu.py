"""Multi-iteration design trajectories of the BASELINE configs on the device path,
against runs of the real reference (tests/golden/make_golden.py --long ...).

These pin the headline fast path (k10 level stencils, single-launch V-cycle
bottom, fp64 defect correction, cooperative OC search) over many design
iterations, not just the first one.

The design loop is chaotic: the reference run at solver_tol 1e-7 instead of
1e-6 (tests/golden/traj_*_tol*.npz, same script; also 3e-7 and 1e-8 for C1 and
the flat case) leaves its own 1e-6 trajectory by > 1e-3 in g from iteration 100
of C1, 26 of C2 and 95 of the flat case, and converges up to 9 iterations (flat)
apart.  No implementation whose solves are not bit-identical to the reference can
track it further than that.
Gates, per iteration k:
  * before the onset k0 (first k where one of the reference's own re-runs differs
    by > 1e-4 in g): g within 1e-3 relative, |dV| <= 1e-4, V* within 1e-4,
    homogenized tensor within max(1e-5, 3x the reference's own deviation) of
    ||kappa||;
  * from k0 on, where the separation is a random walk whose timing no second
    run reproduces: the median and the maximum of |dg| / g and |dV| within 3x
    those of the reference's own deviation (floors 1e-3 and 1e-4);
  * runs to convergence: converged, final g <= 1e-4, the convergence iteration
    within max(5, 2 x the reference's own shift) and the final volume within
    max(1e-3, 2 x the reference's own shift);
  * the 2-D case (an OC tie at its third update, see its test): the ensemble of
    runs at the reference's 8 solver tolerances against the reference's 8 runs.
"""

import numpy as np
import pytest

from otm_testutil import cuda_available, golden

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def otm():
    import paper_2405_19991_b200 as m
    return m


def _run(otm, g, max_iter=None):
    dims = tuple(int(d) for d in g["dims"])
    target = otm.ObjectiveSpec("mse", otm.ConductivityTensor(np.asarray(g["target"], float)))
    cfg = otm.RunConfig(dims=dims, target=target, filter=otm.FilterSpec(float(g["filter_radius"])),
                        init=otm.InitPattern("iwp", float(g["vf"]), seed=0),
                        max_iter=int(max_iter or g["max_iter"]))
    kap = []
    res = otm.run_optimization(cfg, callback=lambda it, fld, r, gv: kap.append(np.array(r.tensor.vec)))
    return res, np.array(kap)


def _envelope(name, g, n):
    """The reference's own per-iteration deviation when its solver tolerance moves
    (every tests/golden/<name>_tol*.npz run: 1e-7, 3e-7, 1e-8), maximum over them."""
    import glob
    import os
    from otm_testutil import GOLDEN
    runs = [np.load(f) for f in sorted(glob.glob(os.path.join(GOLDEN, name.replace(".npz", "_tol*.npz"))))]
    if not runs:
        return None
    m = min([n, len(g["g"])] + [len(p["g"]) for p in runs])
    kn = np.linalg.norm(np.nan_to_num(g["kappa"][:m]), axis=1)
    eg = np.max([np.abs(g["g"][:m] - p["g"][:m]) / np.abs(g["g"][:m]) for p in runs], axis=0)
    ev = np.max([np.abs(g["volfrac"][:m] - p["volfrac"][:m]) for p in runs], axis=0)
    ek = np.maximum.accumulate(np.max([np.nanmax(np.abs(g["kappa"][:m] - p["kappa"][:m]), axis=1) / kn
                                       for p in runs], axis=0))
    dn = max(abs(int(p["iterations"]) - int(g["iterations"])) for p in runs)
    dV = max(abs(float(p["volfrac"][-1]) - float(g["volfrac"][-1])) for p in runs)
    return (dn, dV), eg, ev, ek


def _compare(res, kap, g, n, env=None):
    gs = np.array([r.g for r in res.log[:n]])
    vs = np.array([r.volfrac for r in res.log[:n]])
    vst = np.array([r.vstar for r in res.log[:n]])
    relg = np.abs(gs - g["g"][:n]) / np.abs(g["g"][:n])
    dv = np.abs(vs - g["volfrac"][:n])
    k0 = n
    tol_k = np.full(k0, 1e-5)
    if env is not None:
        _, eg, ev, ek = env
        over = np.nonzero(eg > 1e-4)[0]
        k0 = min(n, int(over[0]) if len(over) else len(eg))
        tol_k = np.maximum(1e-5, 3.0 * ek[:k0])
    # strict window
    assert relg[:k0].max() <= 1e-3, ("g", int(relg[:k0].argmax()), float(relg[:k0].max()))
    assert dv[:k0].max() <= 1e-4, ("volume", int(dv[:k0].argmax()), float(dv[:k0].max()))
    assert np.abs(vst[:k0] - g["vstar"][:k0]).max() <= 1e-4
    ref_k = g["kappa"][:k0]
    finite = np.isfinite(ref_k)
    kerr = np.abs(np.where(finite, kap[:k0] - ref_k, 0.0)).max(axis=1) / np.linalg.norm(
        np.where(finite, ref_k, 0.0), axis=1)
    assert (kerr <= tol_k[:k0]).all(), ("tensor", int(np.argmax(kerr > tol_k[:k0])), float(kerr.max()))
    # past the onset the separation is a random walk whose timing no second run
    # reproduces; what must agree is its size: median and maximum of our deviation
    # within 3x those of the reference's own (floors 1e-3 in g, 1e-4 in V)
    if k0 < n:
        _, eg, ev, _ = env
        m = min(n, len(eg))
        for ours, theirs, floor, what in ((relg[k0:m], eg[k0:m], 1e-3, "g"), (dv[k0:m], ev[k0:m], 1e-4, "volume")):
            assert np.median(ours) <= 3.0 * np.median(theirs) + floor, (what, "median", float(np.median(ours)),
                                                                      float(np.median(theirs)))
            assert ours.max() <= 3.0 * theirs.max() + floor, (what, "max", float(ours.max()), float(theirs.max()))
    return k0


def _converged_like_reference(res, g, env):
    n_ref = int(g["iterations"])
    assert res.converged
    assert res.log[-1].g <= 1e-4
    dn, dV = env[0] if env is not None else (0, 0.0)
    assert abs(len(res.log) - n_ref) <= max(5, 2 * dn), (len(res.log), n_ref, dn)
    assert abs(res.field.mean() - float(g["volfrac"][-1])) <= max(1e-3, 2 * dV)


def test_c2_64_cubed_30_iterations(otm):
    """Config 2 (64^3 orthotropic, vf 0.5): 30 design iterations, k10 path at level 0."""
    g = golden("traj_c2_30.npz")
    res, kap = _run(otm, g)
    assert len(res.log) == 30
    _compare(res, kap, g, 30, _envelope("traj_c2_30.npz", g, 30))


@pytest.mark.parametrize("name", ["traj_c3_3.npz", "traj_c3_10.npz"])
def test_c3_128_cubed_trajectory(otm, name):
    """Config 3 (the headline 128^3 fully anisotropic design): the first design
    iterations of the benchmarked run against the reference."""
    try:
        g = golden(name)
    except FileNotFoundError:
        pytest.skip(f"{name} not generated")
    res, kap = _run(otm, g)
    n = int(g["iterations"])
    assert len(res.log) == n
    _compare(res, kap, g, n)


def test_c4_256_cubed_two_iterations(otm):
    """Config 4 (256^3, the C3 target): the first two design iterations against the
    reference -- the level stencils on nz = 256 and, beyond the L2, the lockstep tile
    order of the k10 march and of the fp64 defect kernel."""
    try:
        g = golden("traj_c4_2.npz")
    except FileNotFoundError:
        pytest.skip("traj_c4_2.npz not generated")
    res, kap = _run(otm, g)
    assert len(res.log) == int(g["iterations"])
    _compare(res, kap, g, int(g["iterations"]))


def test_c1_to_convergence(otm):
    """Config 1 (32^3 isotropic, vf 0.3) run to convergence: the reference stops at
    iteration 237 with g 9.98e-5 and V 0.2335 (tests/test_acceptance.py:171-179)."""
    g = golden("traj_c1_conv.npz")
    res, kap = _run(otm, g)
    env = _envelope("traj_c1_conv.npz", g, len(g["g"]))
    _converged_like_reference(res, g, env)
    _compare(res, kap, g, min(len(res.log), int(g["iterations"])), env)


def test_flat_100x100x1_to_convergence(otm):
    """The reference's 2-D acceptance case (tests/test_acceptance.py:144-158):
    100x100x1 grid, filter radius 2, NaN-masked target components, to g <= 1e-4.

    On this grid the OC moves are quantised (0.02 / 10^4 per element) and the
    update 2 -> 3 is a tie of the bisection's stopping rule: the free-step mean
    exceeds the volume bound by the bisection tolerance 1e-5 to within 5e-17
    (optimize.py:141-158), so the side it falls on is decided by the last bit of a
    sum (the reference's own oc_update, given this run's iteration-2 state, lands
    where this run does).  Iterations 1-2 are compared strictly; where the run ends is
    checked against the reference's ensemble in test_flat_100x100x1_ensemble."""
    g = golden("traj_flat100.npz")
    res, kap = _run(otm, g)
    assert res.converged and res.log[-1].g <= 1e-4
    _compare(res, kap, g, 2)


def test_flat_100x100x1_ensemble(otm):
    """Where the 2-D run ends is chaotic: the reference's own runs at solver_tol 2e-6 ..
    1e-8 (tests/golden/traj_flat100*.npz, 8 runs) converge after 289-338 iterations at
    volume 0.5203-0.5223.  The same 8 tolerances here: every run converges (g <= 1e-4,
    also at 1e-8, where the fp32 breakdown guard restarts stalled inner solves), the
    iteration counts lie inside the reference's range widened by its own spread, and
    the median final volume lies inside the reference's range (+-1e-3)."""
    import glob
    import os
    from otm_testutil import GOLDEN
    refs = {}
    for f in glob.glob(os.path.join(GOLDEN, "traj_flat100*.npz")):
        tag = os.path.basename(f)[len("traj_flat100"):-4]
        refs[float(tag[4:]) if tag else 1e-6] = np.load(f)
    assert len(refs) >= 8
    n_ref = np.array([int(p["iterations"]) for p in refs.values()])
    v_ref = np.array([float(p["volfrac"][-1]) for p in refs.values()])
    spread = int(n_ref.max() - n_ref.min())
    g0 = refs[1e-6]
    its, vols = [], []
    for tol in sorted(refs):
        dims = tuple(int(d) for d in g0["dims"])
        cfg = otm.RunConfig(dims=dims, target=otm.ObjectiveSpec("mse", otm.ConductivityTensor(
            np.asarray(g0["target"], float))), filter=otm.FilterSpec(float(g0["filter_radius"])),
            init=otm.InitPattern("iwp", float(g0["vf"]), seed=0), max_iter=int(g0["max_iter"]),
            solver_tol=tol)
        res = otm.run_optimization(cfg)
        assert res.converged and res.log[-1].g <= 1e-4, (tol, res.log[-1].g)
        its.append(len(res.log))
        vols.append(float(res.field.mean()))
    assert n_ref.min() - spread <= min(its) and max(its) <= n_ref.max() + spread, (its, n_ref)
    assert v_ref.min() - 1e-3 <= np.median(vols) <= v_ref.max() + 1e-3, (vols, v_ref)
