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
                                        ((64, 32, 32), 4), ((16, 16, 16), 2)])
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
