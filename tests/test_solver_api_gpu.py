"""The reference's solver-level API on the device (solver.py:66-406): level arrays,
per-level factors, relax_gs8, restrict, prolong_correct, coarse_solve,
GridHierarchy.vcycle, apply_K on coarse levels, residual_history and the
per-case V-cycle budget -- against the CPU oracle (oracle/otm_oracle.py, pinned
to the reference by tests/test_oracle_golden.py), the reference's golden
vectors and the properties the reference's own tests check
(tests/test_solver.py:127-226, 322-361 of the reference).
"""

import numpy as np
import pytest

from otm_testutil import cuda_available, golden

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

GRIDS = [(8, 8, 8), (16, 8, 4), (12, 12, 1), (8, 4, 2), (16, 16, 16)]


@pytest.fixture(scope="module")
def otm():
    import paper_2405_19991_b200 as m
    return m


@pytest.fixture(scope="module")
def O():
    from oracle import otm_oracle
    return otm_oracle


def _pair(otm, O, dims, seed=0, lo=0.05):
    kap = np.random.default_rng(seed).uniform(lo, 1.0, dims)
    h = otm.GridHierarchy(dims, dtype="float64")
    h.build(kap)
    ho = O.Hierarchy(dims)
    ho.build(kap)
    return h, ho, kap


@pytest.mark.parametrize("dims", GRIDS)
def test_level_factors_and_operator(otm, O, dims):
    h, ho, _ = _pair(otm, O, dims, 1)
    assert [lv.dims for lv in h.levels] == [lv.dims for lv in ho.levels]
    rng = np.random.default_rng(2)
    for lv, lo in zip(h.levels, ho.levels):
        assert np.array_equal(lv.kappa, lo.kappa)            # child means, same op order
        T = rng.standard_normal(lv.dims)
        got = otm.apply_K(lv, T)
        want = lo.apply(T)
        assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


def test_level_kappa_matches_reference_golden(otm):
    g = golden("operator.npz")
    h = otm.GridHierarchy((16, 16, 16), dtype="float64")
    h.build(g["chain_kappa16"])
    for li, lv in enumerate(h.levels):
        assert np.array_equal(lv.kappa, g[f"chain_level{li}_kappa"]), li
        assert np.allclose(lv.template, g[f"chain_level{li}_template"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("dims", GRIDS)
def test_relax_gs8_matches_oracle(otm, O, dims):
    h, ho, _ = _pair(otm, O, dims, 3)
    rng = np.random.default_rng(4)
    for li in range(len(h.levels)):
        lv, lo = h.levels[li], ho.levels[li]
        if any(n > 1 and n % 2 for n in lv.dims):
            continue
        f = rng.standard_normal(lv.dims)
        T = rng.standard_normal(lv.dims)
        lv.f[...] = f
        lv.T[...] = T
        lo.f[...] = f
        lo.T[...] = T
        otm.relax_gs8(lv, sweeps=2)
        O.gauss_seidel8(lo, 2)
        assert np.abs(lv.T - lo.T).max() <= 1e-12 * np.abs(lo.T).max()


def test_relax_fixed_point_and_odd_axes(otm, O):
    """tests/test_solver.py:144-173 of the reference."""
    rng = np.random.default_rng(6)
    kappa = rng.uniform(0.2, 1, (4, 4, 4))
    h = otm.GridHierarchy((4, 4, 4), dtype="float64")
    h.build(kappa)
    ho = O.Hierarchy((4, 4, 4))
    ho.build(kappa)
    x = rng.standard_normal((4, 4, 4))
    x -= x.mean()
    lev = h.levels[0]
    lev.f[...] = ho.levels[0].apply(x)
    lev.T[...] = x
    otm.relax_gs8(lev, sweeps=1)
    assert np.allclose(lev.T, x, atol=1e-11)
    h8 = otm.GridHierarchy((8, 8, 8), dtype="float64")
    h8.build(np.ones((8, 8, 8)))
    lv = h8.levels[0]
    f = rng.standard_normal((8, 8, 8))
    lv.f[...] = f - f.mean()
    lv.T[...] = 0
    r0 = np.linalg.norm(lv.f - otm.apply_K(lv, lv.T))
    otm.relax_gs8(lv, sweeps=10)
    assert np.linalg.norm(lv.f - otm.apply_K(lv, lv.T)) < r0
    hodd = otm.GridHierarchy((5, 4, 4), dtype="float64")
    hodd.build(np.full((5, 4, 4), 0.5))
    with pytest.raises(ValueError):
        otm.relax_gs8(hodd.levels[0], 1)


@pytest.mark.parametrize("dims", GRIDS)
def test_transfer_matches_oracle_and_adjoint(otm, O, dims):
    h, ho, _ = _pair(otm, O, dims, 7)
    if len(h.levels) < 2:
        pytest.skip("single level")
    rng = np.random.default_rng(8)
    a = rng.standard_normal(h.levels[0].dims)
    b = rng.standard_normal(h.levels[1].dims)
    h.levels[0].r[...] = a
    otm.restrict(h.levels[0], h.levels[1])
    ho.levels[0].r[...] = a
    O.restrict_fw(ho.levels[0], ho.levels[1])
    assert np.abs(h.levels[1].f - ho.levels[1].f).max() <= 1e-14 * np.abs(a).max()
    Ra = h.levels[1].f.copy()
    h.levels[1].T[...] = b
    h.levels[0].T[...] = 0
    otm.prolong_correct(h.levels[0], h.levels[1])
    ho.levels[1].T[...] = b
    ho.levels[0].T[...] = 0
    O.prolong_add(ho.levels[0], ho.levels[1])
    assert np.abs(h.levels[0].T - ho.levels[0].T).max() <= 1e-14 * np.abs(b).max()
    # R = P^T / 2^(coarsened axes)  (reference tests/test_solver.py:190-204)
    ncoarse = sum(c < f for c, f in zip(h.levels[1].dims, h.levels[0].dims))
    lhs = float((Ra * b).sum())
    rhs = float((a * h.levels[0].T).sum())
    assert lhs == pytest.approx(rhs / 2 ** ncoarse, rel=1e-10)


@pytest.mark.parametrize("dims", [(4, 4, 4), (8, 8, 8), (12, 12, 1), (100, 100, 1)])
def test_coarse_solve(otm, O, dims):
    h, ho, _ = _pair(otm, O, dims, 9, lo=0.1)
    lev, lo = h.levels[-1], ho.levels[-1]
    f = np.random.default_rng(10).standard_normal(lev.dims)
    f -= f.mean()
    lev.f[...] = f
    T = otm.coarse_solve(h)
    lo.f[...] = f
    ho.coarse()
    assert np.abs(T - lo.T).max() <= 1e-9 * np.abs(lo.T).max()
    res = np.linalg.norm(lo.apply(T) - f) / np.linalg.norm(f)
    assert res < 1e-10
    assert abs(T.mean()) < 1e-12
    lev.f[...] = 1.0 + f
    with pytest.warns(RuntimeWarning):
        otm.coarse_solve(h)
    lev.f[...] = 0.0
    assert np.abs(otm.coarse_solve(h)).max() == 0


@pytest.mark.parametrize("dims", [(16, 16, 16), (16, 8, 4), (12, 12, 1)])
def test_vcycle_matches_oracle(otm, O, dims):
    """GridHierarchy.vcycle: the reference's GS-8 V-cycle (solver.py:326-338)."""
    h, ho, _ = _pair(otm, O, dims, 11)
    rng = np.random.default_rng(12)
    f = rng.standard_normal(dims)
    f -= f.mean()
    T = rng.standard_normal(dims) * 0.1
    h.levels[0].f[...] = f
    h.levels[0].T[...] = T
    ho.levels[0].f[...] = f
    ho.levels[0].T[...] = T
    for _ in range(3):
        h.vcycle()
        ho.vcycle()
    for lv, lo in zip(h.levels, ho.levels):
        assert np.abs(lv.T - lo.T).max() <= 1e-10 * max(1.0, np.abs(lo.T).max())
        assert np.abs(lv.f - lo.f).max() <= 1e-10 * max(1.0, np.abs(lo.f).max())


def test_residual_history_and_contraction(otm):
    """One entry per V-cycle, decreasing to tol; mean contraction <= 0.7 on SIMP
    fields (reference tests/test_solver.py:322-335)."""
    rng = np.random.default_rng(17)
    mp = otm.MaterialParams()
    worst = 0.0
    for _ in range(3):
        rho = rng.uniform(0.1, 1.0, (16, 16, 16))
        h = otm.GridHierarchy((16, 16, 16), dtype="float64")
        h.build(otm.simp_conductivity(rho, mp))
        f = otm.assemble_macro_load(h, 0)
        T, cycles = otm.solve_equation(h, f, tol=1e-9, max_vcycles=100)
        res = np.asarray(h.residual_history)
        assert len(res) == cycles
        assert res[-1] <= 1e-9
        ratios = res[1:] / res[:-1]
        worst = max(worst, float(ratios.mean()))
    assert worst <= 0.7, worst
    T, cycles = otm.solve_equation(h, np.zeros((16, 16, 16)))
    assert cycles == 0 and h.residual_history == []


def test_max_vcycles_is_per_case(otm):
    """Each load case has its own budget of max_vcycles (homogenize.py:85-90 runs
    three solves): the smallest budget that succeeds is below the total V-cycle
    count of the three cases, which a shared budget could never allow."""
    rng = np.random.default_rng(21)
    rho = rng.uniform(0.05, 1.0, (16, 16, 16))
    mp = otm.MaterialParams()
    h = otm.GridHierarchy((16, 16, 16), dtype="float64")
    _, total = otm.solve_cases(h, rho, mp, tol=1e-8)
    ok = []
    for budget in range(total // 3, total + 1):
        try:
            otm.solve_cases(h, rho, mp, tol=1e-8, max_vcycles=budget)
            ok.append(budget)
            break
        except otm.ConvergenceError:
            pass
    assert ok, "no budget up to the total succeeded"
    assert ok[0] < total
    assert ok[0] * 3 >= total


def test_flat_grid_solve_vs_oracle(otm, O):
    """100 x 100 x 1 (reference tests/test_acceptance.py:144-158 grid): the batched
    solve with the flat-axis diagonal."""
    dims = (100, 100, 1)
    rng = np.random.default_rng(5)
    rho = rng.uniform(0.05, 1.0, dims)
    mp = otm.MaterialParams()
    h = otm.GridHierarchy(dims)
    T, cyc = otm.solve_cases(h, rho, mp, tol=1e-9)
    assert cyc < 150, cyc
    ho = O.Hierarchy(dims)
    To, _ = O.solve_three(ho, rho, O.Material(), tol=1e-11)
    for i in range(2):
        assert np.abs(T[i] - To[i]).max() <= 1e-6 * np.abs(To[i]).max()


def test_elem_diff_matches_corner_formula(otm):
    """HomogenizationResult.elem_diff (homogenize.py:94-100) from the device kernel
    against c_a[i] - T_i[e + c_a] evaluated with numpy rolls."""
    from paper_2405_19991_b200.element import CORNERS
    dims = (8, 6, 4)
    rng = np.random.default_rng(11)
    rho_f = rng.uniform(0.1, 1.0, dims)
    mp = otm.MaterialParams()
    h = otm.GridHierarchy(dims)
    T, _ = otm.solve_cases(h, rho_f, mp, tol=1e-10)
    res = otm.effective_tensor(h, T, rho_f, mp)
    w = res.elem_diff
    for i in range(3):
        ref = np.stack([float(CORNERS[a, i]) - np.roll(T[i], tuple(-int(s) for s in CORNERS[a]), axis=(0, 1, 2))
                        for a in range(8)], axis=-1).astype(np.float32)
        assert w[i].shape == dims + (8,)
        assert np.array_equal(w[i], ref)
