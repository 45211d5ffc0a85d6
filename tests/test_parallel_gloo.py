"""Multi-rank slab decomposition on CPU (gloo, world size 2 and 4): the ghost-plane
exchange and the scalar all-reduce reproduce the single-domain operator, loads,
tensor sums and filter of the CPU oracle exactly.  This is the exchange pattern the
multi-GPU solver uses (NCCL instead of gloo)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_19991_b200.parallel import (SlabPlan, allreduce_sum, gather_level, halo_exchange, level_dims,
                                            owned_part, with_ghosts)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, dims, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import otm_oracle as O
        rng = np.random.default_rng(seed)
        kap = rng.uniform(1e-4, 1.0, dims)
        T = rng.standard_normal(dims)
        rho = rng.uniform(0.0, 1.0, dims)
        plan = SlabPlan(dims, world, rank)
        lev = plan.levels[0]
        # each rank only ever sees its own slab; ghosts come from the exchange
        kap_p = halo_exchange(with_ghosts(torch.from_numpy(kap[lev.x0:lev.x1].copy())), plan).numpy()
        T_p = halo_exchange(with_ghosts(torch.from_numpy(T[lev.x0:lev.x1].copy())), plan).numpy()
        rho_p = halo_exchange(with_ghosts(torch.from_numpy(rho[lev.x0:lev.x1].copy())), plan).numpy()
        # operator and loads on the padded slab (the oracle wraps x periodically, which only
        # touches the ghost planes whose results are discarded)
        hp = O.Hierarchy(kap_p.shape, coarse_target=10 ** 9)
        hp.build(kap_p)
        KT_local = hp.levels[0].apply(T_p)[1:-1]
        f_local = np.stack([O.macro_load(hp, i)[1:-1] for i in range(3)])
        filt_local = O.filter_fwd(rho_p)[1:-1]
        # a global scalar: sum of kappa * (K T) over owned vertices, all-reduced
        s = allreduce_sum(torch.tensor([float((kap[lev.x0:lev.x1] * KT_local).sum())], dtype=torch.float64))
        full_KT = gather_level(torch.from_numpy(np.ascontiguousarray(KT_local)), plan).numpy()
        q.put((rank, KT_local, f_local, filt_local, float(s[0]), full_KT, (lev.x0, lev.x1)))
    finally:
        dist.destroy_process_group()


def _run(world, dims, seed=0):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


@pytest.mark.parametrize("world,dims", [(2, (8, 6, 4)), (4, (16, 4, 6))])
def test_slab_exchange_reproduces_single_domain(world, dims):
    from oracle import otm_oracle as O
    res = _run(world, dims)
    rng = np.random.default_rng(0)
    kap = rng.uniform(1e-4, 1.0, dims)
    T = rng.standard_normal(dims)
    rho = rng.uniform(0.0, 1.0, dims)
    h = O.Hierarchy(dims, coarse_target=10 ** 9)
    h.build(kap)
    KT = h.levels[0].apply(T)
    f = np.stack([O.macro_load(h, i) for i in range(3)])
    filt = O.filter_fwd(rho)
    total = float((kap * KT).sum())
    for rank, KT_l, f_l, filt_l, s, full_KT, (x0, x1) in res:
        assert np.abs(KT_l - KT[x0:x1]).max() <= 1e-13 * np.abs(KT).max()
        assert np.abs(f_l - f[:, x0:x1]).max() <= 1e-15
        assert np.array_equal(filt_l, filt[x0:x1])          # same tap order -> bit-exact
        assert s == pytest.approx(total, rel=1e-12)
        assert np.abs(full_KT - KT).max() <= 1e-13 * np.abs(KT).max()


def test_plan_levels_and_agglomeration():
    p = SlabPlan((256, 256, 256), 8, 3)
    dims = [l.dims for l in p.levels]
    assert dims == level_dims((256, 256, 256))
    # 256/8 = 32 planes at level 0 ... 2 planes at 16^3, then agglomerate at 8^3
    assert [l.distributed for l in p.levels] == [True, True, True, True, True, False, False]
    assert p.levels[0].x0 == 96 and p.levels[0].x1 == 128
    assert p.levels[3].x0 == 12 and p.levels[3].x1 == 16
    assert p.agglomeration_level == 5
    # weak-scaling shape of BASELINE config 5 on 8 GPUs
    p5 = SlabPlan((512, 512, 512), 8, 0)
    assert p5.levels[0].nx_local == 64 and p5.agglomeration_level == 6
    with pytest.raises(ValueError):
        SlabPlan((6, 6, 6), 4, 0)


def test_owned_part_single_rank():
    plan = SlabPlan((8, 4, 4), 1, 0)
    full = torch.arange(8 * 16, dtype=torch.float64).reshape(8, 4, 4)
    assert torch.equal(owned_part(full, plan), full)
    pad = halo_exchange(with_ghosts(full), plan)
    assert torch.equal(pad[0], full[-1]) and torch.equal(pad[-1], full[0])
