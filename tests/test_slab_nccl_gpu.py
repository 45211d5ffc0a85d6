"""The slab path across processes over NCCL (DistComm + CudaSlabBackend, one GPU per
rank, world size 2): the distributed solve and tensor against the single-GPU
solver on the same density.  Needs >= 2 GPUs; skipped otherwise (the build boxes
of this project have one), the same orchestration is covered over gloo on CPU by
tests/test_slab_gloo.py and on one GPU with in-process slabs by
tests/test_slab_gpu.py."""

import os
import socket

import numpy as np
import pytest

from otm_testutil import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, out_path):
    import torch
    import torch.distributed as dist

    import paper_2405_19991_b200 as otm
    from paper_2405_19991_b200.slab import CudaSlabBackend, DistComm, SlabSolver

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    rng = np.random.default_rng(3)
    rho = rng.uniform(0.05, 1.0, dims)
    mp = otm.MaterialParams()
    kap = otm.simp_conductivity(rho, mp)
    nxl = dims[0] // world
    backend = CudaSlabBackend(3 * (nxl + 2) * dims[1] * dims[2])
    solver = SlabSolver(dims, DistComm(), backend)
    solver.build_kappa([torch.from_numpy(np.ascontiguousarray(kap[rank * nxl:(rank + 1) * nxl])).cuda()])
    solver.solve(tol=1e-9)
    kh = solver.tensor()
    T = solver.fields()
    if rank == 0:
        h = otm.GridHierarchy(dims)
        h.build(kap)
        T1, _, _ = h.solve3(None, tol=1e-9)
        import ctypes as C
        k1 = (C.c_double * 6)()
        h.ctx.call("otm_tensor", k1)
        err_T = float((T.double() - T1).abs().max() / T1.abs().max())
        err_k = float(np.abs(np.array(kh) - np.array(k1[:])).max() / np.linalg.norm(k1[:]))
        np.save(out_path, np.array([err_T, err_k]))
    dist.barrier()
    dist.destroy_process_group()


def test_slab_solve_over_nccl_matches_single_gpu(tmp_path):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (NCCL across processes)")
    dims = (64, 64, 64)
    out = str(tmp_path / "err.npy")
    mp.spawn(_worker, args=(2, _free_port(), dims, out), nprocs=2, join=True)
    err_T, err_k = np.load(out)
    assert err_T <= 1e-6, err_T
    assert err_k <= 1e-9, err_k
