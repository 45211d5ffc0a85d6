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


@pytest.mark.parametrize("dims,world", [((32, 32, 32), 2), ((64, 64, 64), 4), ((16, 32, 128), 2), ((8, 16, 16), 4)])
def test_slab_solve_halo_overlap_split(dims, world, monkeypatch):
    """OTM_SLAB_OVERLAP=1: every stencil after a halo exchange runs as the interior
    output planes [2, nxl) + planes 1 and nxl (otm_slab_stencil_range; k10 ranges of
    one plane at nz 64 / 128) with the three partial dot products added -- what the
    NCCL path does between processes.  Same answers as the whole-slab launches."""
    import paper_2405_19991_b200 as otm
    rng = np.random.default_rng(7 + world)
    rho_f = rng.uniform(0.05, 1.0, dims)
    mp = otm.MaterialParams()
    h = otm.GridHierarchy(dims)
    T_ref, _ = otm.solve_cases(h, rho_f, mp, tol=1e-10)
    base, cyc0 = _solve_slabs(dims, world, rho_f, tol=1e-10)
    monkeypatch.setenv("OTM_SLAB_OVERLAP", "1")
    split, cyc1 = _solve_slabs(dims, world, rho_f, tol=1e-10)
    assert split.overlap and not base.overlap
    T0 = base.fields().cpu().numpy()
    T1 = split.fields().cpu().numpy()
    for i in range(3):
        assert np.abs(T1[i] - T_ref[i]).max() <= 1e-7 * np.abs(T_ref[i]).max()
        assert np.abs(T1[i] - T0[i]).max() <= 1e-7 * np.abs(T0[i]).max()
    assert abs(cyc1 - cyc0) <= 3


def test_stencil_range_writes_only_its_planes():
    """otm_slab_stencil_range on [lo, hi) equals the whole-slab launch on those planes
    (bit for bit: the same per-vertex arithmetic) and leaves the other planes alone;
    the range dot products add up to the whole-slab ones."""
    import torch
    from paper_2405_19991_b200.slab import CudaSlabBackend
    for dims in ((6, 16, 16), (6, 64, 64)):        # generic kernel / k10 march
        nxl, ny, nz = dims
        B = CudaSlabBackend(3 * (nxl + 2) * ny * nz)
        g = torch.Generator().manual_seed(5)
        kap = (0.05 + torch.rand((nxl + 2, ny, nz), generator=g)).cuda()
        dinv = (0.5 + torch.rand((nxl + 2, ny, nz), generator=g)).cuda()
        a = torch.randn((3, nxl + 2, ny, nz), generator=g).cuda()
        f = torch.randn((3, nxl + 2, ny, nz), generator=g).cuda()
        sc = (1.0, 1.0, 1.0)
        for op in (0, 1, 2):
            o1 = torch.zeros_like(a)
            o2 = torch.zeros_like(a) if op == 0 else None
            B.stencil(op, dims, sc, kap, a if op else None, f if op < 2 else None, dinv if op < 2 else None, 0.9,
                      o1, o2)
            whole = B.stencil_dev(op, dims, sc, kap, a if op else None, f if op < 2 else None,
                                  dinv if op < 2 else None, 0.9, torch.zeros_like(a)) if op else None
            tot = 0.0
            r1 = torch.full_like(a, 7.0)
            r2 = torch.full_like(a, 7.0) if op == 0 else None
            for lo, hi in ((2, nxl), (1, 2), (nxl, nxl + 1)):
                d = B.stencil_range(op, dims, sc, kap, a if op else None, f if op < 2 else None,
                                    dinv if op < 2 else None, 0.9, r1, r2, lo, hi, want_dots=op > 0)
                if op:
                    tot = tot + d
            assert torch.equal(r1[:, 1:nxl + 1], o1[:, 1:nxl + 1])
            assert (r1[:, 0] == 7.0).all() and (r1[:, nxl + 1] == 7.0).all()
            if op == 0:
                assert torch.equal(r2[:, 1:nxl + 1], o2[:, 1:nxl + 1])
            else:
                assert torch.allclose(tot, whole, rtol=1e-12, atol=0)


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
