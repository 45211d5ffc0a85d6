"""Slab-decomposed solve on the device (include/otm_slab.h kernels): 1, 2 and 4 slabs
of one grid held in one process (LocalComm: halo exchange = plane copies, scalar
all-reduce = fixed-order sum), against the single-GPU solver and the CPU oracle.
The multi-process transport (DistComm over torch.distributed) is covered with gloo
in tests/test_slab_gloo.py."""

import numpy as np
import pytest

from otm_testutil import cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


def _solve_slabs(dims, world, rho_f, tol):
    import torch
    from paper_2405_19991_b200.slab import CudaSlabBackend, LocalComm, SlabSolver
    comm = LocalComm(world)
    solver = SlabSolver(dims, comm, CudaSlabBackend(3 * int(np.prod(dims))))
    nxl = dims[0] // world
    parts = [torch.from_numpy(np.ascontiguousarray(rho_f[r * nxl:(r + 1) * nxl])).cuda() for r in range(world)]
    solver.build_density(parts)
    cycles = solver.solve(tol=tol)
    return solver, cycles


@pytest.mark.parametrize("dims,world", [((32, 32, 32), 1), ((32, 32, 32), 2), ((32, 32, 32), 4),
                                        ((64, 32, 32), 4), ((16, 16, 16), 2),
                                        # nz = 64 / 128: the slab stencils run the k10 march on the
                                        # interior planes (launch_k10_range)
                                        ((32, 64, 64), 2), ((64, 64, 64), 4), ((16, 32, 128), 2)])
def test_slab_solve_matches_single_gpu(dims, world):
    import paper_2405_19991_b200 as otm
    rng = np.random.default_rng(world + dims[0])
    rho_f = rng.uniform(0.05, 1.0, dims)
    mp = otm.MaterialParams()
    h = otm.GridHierarchy(dims)
    T_ref, _ = otm.solve_cases(h, rho_f, mp, tol=1e-10)
    k_ref = otm.effective_tensor(h, T_ref, rho_f, mp).tensor.vec
    solver, cycles = _solve_slabs(dims, world, rho_f, tol=1e-10)
    T = solver.fields().cpu().numpy()
    for i in range(3):
        assert np.abs(T[i] - T_ref[i]).max() <= 1e-7 * np.abs(T_ref[i]).max()
    k = solver.tensor()
    assert np.abs(k - k_ref).max() <= 1e-9 * np.linalg.norm(k_ref)
    assert cycles > 0


def test_slab_design_run_tracks_single_gpu():
    """12 OC iterations of the slab design loop (2 slabs) against run_optimization."""
    import torch
    import paper_2405_19991_b200 as otm
    from paper_2405_19991_b200.slab import CudaSlabBackend, LocalComm, SlabDesignRun
    dims = (32, 32, 32)
    target = otm.ObjectiveSpec("mse", otm.ConductivityTensor([0.1, 0.1, 0.1, 0, 0, 0]))
    cfg = otm.RunConfig(dims=dims, target=target, init=otm.InitPattern("iwp", 0.3, seed=0), max_iter=12,
                        conv_threshold=0.0, solver_tol=1e-10)
    ref = otm.run_optimization(cfg)
    seed = otm.init_density(dims, cfg.init).rho
    W = 2
    nxl = dims[0] // W
    run = SlabDesignRun(cfg, LocalComm(W), CudaSlabBackend(3 * int(np.prod(dims))),
                        [torch.from_numpy(np.ascontiguousarray(seed[r * nxl:(r + 1) * nxl])).cuda() for r in range(W)])
    while not run.finished:
        run.step()
    assert len(run.log) == len(ref.log) == 12
    for a, b in zip(run.log, ref.log):
        assert abs(a.g - b.g) <= 1e-6 * max(abs(b.g), 1e-12)
        assert abs(a.volfrac - b.volfrac) <= 1e-9
    rho = run.density().cpu().numpy()
    assert np.abs(rho - ref.field.rho).max() <= 1e-6
