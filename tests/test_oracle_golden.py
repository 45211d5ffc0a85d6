"""Pin the CPU oracle against golden vectors produced by the real reference.

The vectors come from tests/golden/make_golden.py (run in the build container
against /root/reference).  If these pass, the oracle is a trustworthy checker
for the CUDA path.
"""

import numpy as np
import pytest

from oracle import otm_oracle as O
from otm_testutil import golden


def test_element_templates():
    g = golden("element.npz")
    assert np.abs(O.K0 - g["K0"]).max() < 1e-15
    assert np.abs(O.F0 - g["f0"]).max() < 1e-15
    # closed-form entries
    assert O.K0[0, 0] == pytest.approx(1 / 3)
    assert O.K0[0, 1] == pytest.approx(0.0, abs=1e-16)
    assert O.K0[0, 3] == pytest.approx(-1 / 12)


@pytest.mark.parametrize("radius,tag", [(1.5, "1p5"), (2.0, "2p0")])
def test_filter(radius, tag):
    g = golden("filter.npz")
    offs, w = O.filter_taps(radius)
    assert np.array_equal(offs, g[f"offs_{tag}"])
    assert np.abs(w - g[f"w_{tag}"]).max() < 1e-16
    assert np.abs(O.filter_fwd(g["rho"], radius) - g[f"fwd_{tag}"]).max() < 1e-15
    assert np.abs(O.filter_adj(g["g"], radius) - g[f"bwd_{tag}"]).max() < 1e-14


def test_symmetry_projection():
    g = golden("filter.npz")
    assert np.array_equal(O.central_symmetrize(g["sym_in"]), g["sym_out"])


@pytest.mark.parametrize("tag", ["a", "b", "c", "d"])
def test_operator_and_load(tag):
    g = golden("operator.npz")
    kap = g[f"kappa_{tag}"]
    h = O.Hierarchy(kap.shape)
    h.build(kap)
    KT = h.levels[0].apply(g[f"T_{tag}"])
    ref = g[f"KT_{tag}"]
    assert np.abs(KT - ref).max() <= 1e-13 * np.abs(ref).max()
    for i in range(3):
        assert np.abs(O.macro_load(h, i) - g[f"f_{tag}"][i]).max() < 1e-14


def test_level_chain_and_child_mean():
    g = golden("operator.npz")
    h = O.Hierarchy((16, 16, 16))
    h.build(g["chain_kappa16"])
    for li, lev in enumerate(h.levels):
        assert np.abs(lev.kappa - g[f"chain_level{li}_kappa"]).max() < 1e-15
        assert np.abs(lev.template - g[f"chain_level{li}_template"]).max() < 1e-15
    keys = list(g["chain_dims_keys"])
    for i, k in enumerate(keys):
        dims = tuple(int(x) for x in k.strip("()").split(","))
        got = [d for d, _ in O.level_chain(dims)]
        assert np.array_equal(np.array(got), g[f"chain_dims_{i}"])


def test_uncoarsenable_rejected():
    with pytest.raises(ValueError):
        O.level_chain((63, 63, 63))


def test_solve_matches_reference():
    g = golden("solve.npz")
    h = O.Hierarchy((8, 8, 8))
    h.build(g["kappa"])
    T, cyc = O.solve(h, g["f"], tol=1e-10)
    assert cyc == int(g["cycles"])
    assert np.abs(T - g["T"]).max() < 1e-12 * np.abs(g["T"]).max()
    assert np.allclose(h.history, g["history"], rtol=1e-6)
    T2, cyc2 = O.solve(h, g["f"], tol=1e-10, x0=g["x0"])
    assert cyc2 == int(g["cycles_warm"])
    assert np.abs(T2 - g["T_warm"]).max() < 1e-12 * np.abs(g["T"]).max()


@pytest.mark.parametrize("name", ["homog_rand8.npz", "homog_iwp16.npz", "homog_rand_6x8x10.npz"])
def test_homogenize_and_sensitivity(name):
    g = golden(name)
    mat = O.Material()
    rho_f = O.filter_fwd(g["rho"])
    assert np.abs(rho_f - g["rho_f"]).max() < 1e-15
    h = O.Hierarchy(rho_f.shape)
    Ts, cyc = O.solve_three(h, rho_f, mat, tol=1e-10)
    assert cyc == int(g["vcycles"])
    E = O.pair_energies(Ts)
    kh = O.tensor_from_energies(E, rho_f, mat)
    assert np.abs(kh - g["kappa_h"]).max() < 1e-12
    assert np.abs(E - g["pair_energy"]).max() < 1e-9
    gval, dG = O.objective("mse", g["target"], kh)
    assert gval == pytest.approx(float(g["g"]), rel=1e-10)
    sf = O.sensitivity(E, rho_f, dG, mat)
    assert np.abs(sf - g["sens_f"]).max() <= 1e-9 * np.abs(g["sens_f"]).max()
    s = O.filter_adj(sf)
    assert np.abs(s - g["sens"]).max() <= 1e-9 * np.abs(g["sens"]).max()


def test_oc_update_bitexact():
    g = golden("oc.npz")
    for k in range(int(g["ncases"])):
        p = O.OC(step_limit=float(g[f"step_{k}"]))
        new, info = O.oc_step(g[f"rho_{k}"], g[f"sens_{k}"], float(g[f"bound_{k}"]), p)
        assert info["active"] == bool(g[f"active_{k}"])
        assert info["lam"] == pytest.approx(float(g[f"lam_{k}"]), rel=1e-12)
        assert np.array_equal(new, g[f"new_{k}"])


def test_governor_trace():
    g = golden("oc.npz")
    st = O.Governor()
    rho = g["gov_rho"]
    for gval, row in zip(g["gov_g"], g["gov_trace"]):
        v = O.governor_step(st, float(gval), float(rho.mean()), float((rho ** 3.0).mean()))
        got = [v, st.df, st.gap, st.count, float(st.reduced), st.pending_decrease]
        assert np.allclose(got, row, rtol=1e-14, atol=0)


@pytest.mark.slow
def test_trajectory_c1_first_iterations():
    """First 12 OC iterations of config 1 (32^3 IWP vf 0.3) vs the reference log."""
    g = golden("traj_c1.npz")
    n = 12
    cfg = O.Run(dims=(32, 32, 32), target=list(g["target"]), init=("iwp", float(g["vf"]), 0),
                max_iter=n)
    rho, kh, log, conv = O.optimize(cfg)
    gs = np.array([r.g for r in log])
    assert np.allclose(gs, g["g"][:n], rtol=1e-6)
    assert np.allclose([r.volfrac for r in log], g["volfrac"][:n], atol=1e-10)
    assert [r.vcycles for r in log] == list(g["vcycles"][:n])


def test_seed_patterns_match_reference_volume():
    g = golden("homog_iwp16.npz")
    assert np.array_equal(O.seed_density((16, 16, 16), "iwp", 0.3), g["rho"])
