"""The device-resident design iteration (otm_run_batch: one graph launch per design
iteration, every decision on the device) against the host-driven path
(otm_run_step / otm_run_update, used when a callback needs the host between the
evaluation and the update): bit-identical densities and logs, the same failure
behaviour, fixed-volume and central-symmetry models."""

import numpy as np
import pytest

from otm_testutil import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def otm():
    import paper_2405_19991_b200 as m
    return m


def _cfg(otm, dims, target, vf, max_iter, **kw):
    return otm.RunConfig(dims=dims, target=otm.ObjectiveSpec("mse", otm.ConductivityTensor(target)),
                         init=otm.InitPattern("iwp", vf, seed=0), max_iter=max_iter, **kw)


def _both(otm, cfg):
    """The same run twice on one hierarchy: whole iterations as graph launches
    (DesignRun.run -> otm_run_batch) and host-driven (DesignRun.step ->
    otm_run_step / otm_run_update)."""
    from paper_2405_19991_b200.optimize import DesignRun, _cached_hierarchy
    out = []
    for graph in (True, False):
        run = DesignRun(cfg, hier=_cached_hierarchy(cfg))
        if graph:
            rc = run.run()
        else:
            rc = 0
            while rc == 0 and not run.finished:
                rc, _ = run.step()
        out.append((rc, run, run.rho.cpu().numpy(), list(run.log)))
    return out


def _same(a, b):
    (rca, ra, rhoa, la), (rcb, rb, rhob, lb) = a, b
    assert rca == rcb == 0
    assert len(la) == len(lb)
    assert np.array_equal(rhoa, rhob)
    for x, y in zip(la, lb):
        assert (x.iter, x.g, x.volfrac, x.volfrac_filtered, x.vstar, x.vcycles) == \
               (y.iter, y.g, y.volfrac, y.volfrac_filtered, y.vstar, y.vcycles)
    assert np.array_equal(ra.kappa.vec, rb.kappa.vec)
    assert ra.st.converged == rb.st.converged


@pytest.mark.parametrize("dims,target,vf,iters", [
    ((32, 32, 32), [0.1, 0.1, 0.1, 0, 0, 0], 0.3, 500),                  # C1 to convergence
    ((128, 128, 128), [0.3, 0.2, 0.1, 0.1, 0.05, 0.05], 0.5, 12),         # C3 (k10 path)
    ((16, 16, 32), [0.2, 0.15, 0.1, 0.02, 0, 0], 0.4, 40),
])
def test_graph_path_matches_host_path(otm, dims, target, vf, iters):
    graph, host = _both(otm, _cfg(otm, dims, target, vf, iters))
    _same(graph, host)


def test_graph_path_symmetry_and_fixed_model(otm):
    cfg = _cfg(otm, (16, 16, 16), [0.2, 0.2, 0.2, 0, 0, 0], 0.5, 15, symmetry="central")
    graph, host = _both(otm, cfg)
    _same(graph, host)
    rho = graph[2]
    assert np.array_equal(rho, rho[::-1, ::-1, ::-1])
    cfg = _cfg(otm, (16, 16, 16), [0.2, 0.2, 0.2, 0, 0, 0], 0.5, 15, model="fixed", volume_bound=0.45)
    graph, host = _both(otm, cfg)
    _same(graph, host)
    assert abs(graph[2].mean() - 0.45) < 1e-4


def test_graph_path_solver_failure(otm):
    """A budget too small for the first solve: OptimizationAborted with an empty
    partial log on both paths (optimize.py:295-298)."""
    cfg = _cfg(otm, (16, 16, 16), [0.2, 0.2, 0.2, 0, 0, 0], 0.5, 10, max_vcycles=2)
    for cb in (None, lambda *a: None):
        with pytest.raises(otm.OptimizationAborted) as err:
            otm.run_optimization(cfg, callback=cb)
        assert "solver failed at iteration 1" in str(err.value)
        assert err.value.partial.iterations == 0


def test_graph_path_one_host_wait_per_batch(otm):
    """The graph path synchronises with the host once per batch of iterations."""
    from paper_2405_19991_b200.optimize import DesignRun, _cached_hierarchy
    cfg = _cfg(otm, (64, 64, 64), [0.3, 0.2, 0.1, 0, 0, 0], 0.5, 48, conv_threshold=0.0)
    run = DesignRun(cfg, hier=_cached_hierarchy(cfg))
    rc, recs = run.run_batch(48, batch=16)
    assert rc == 0 and len(recs) == 48 and run.finished
    assert [r.iter for r in recs] == list(range(1, 49))
