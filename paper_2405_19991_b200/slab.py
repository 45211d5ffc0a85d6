"""Slab-decomposed homogenization solve: the multi-GPU path.

The periodic grid is cut along axis 0 (x, the slowest C-order axis of the
reference's (nx, ny, nz) arrays) into one slab per rank.  Every level of the
multigrid hierarchy whose planes still split evenly (>= 2 planes, even count per
rank) is distributed the same way; fields carry one ghost plane per side,
refreshed by a halo exchange with the two neighbouring ranks before every stencil
that reads them.  The global couplings are scalars only: the PCG dot products,
the defect norms, the load and temperature means and the tensor sums, all
all-reduced.  The first level that no longer splits is agglomerated: its
right-hand side is all-gathered and every rank runs the rest of the V-cycle
redundantly with the single-GPU hierarchy (``otm_vcycle``), keeping its own slab
of the correction.

The algorithm is the single-GPU one (fp64 defect correction around an fp32
MG-PCG with a damped-Jacobi V-cycle, solver.py:366-406 semantics for ``tol``), so
a slab solve matches the single-GPU solve to the solver tolerance.

Pieces:
  * ``SlabSolver``   the orchestration, written against a backend and a comm;
  * ``CudaSlabBackend`` the device kernels of include/otm_slab.h (libotm.so);
  * ``DistComm``     one slab per process over torch.distributed (NCCL on GPUs,
                     gloo on CPU), ``LocalComm`` several slabs in one process
                     (single-GPU validation of the slab kernels; no collective).
Tests run the orchestration with a numpy backend under gloo, world size 2
(tests/test_slab_gloo.py), and the CUDA backend on one GPU with 1, 2 and 4
local slabs against the single-GPU solver (tests/test_slab_gpu.py).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np



def level_dims(dims, coarse_target: int = 64):
    """The reference level chain (solver.py:217-231): halve every axis > 1 while the
    level has more than coarse_target vertices and those axes are even."""
    chain = [tuple(int(n) for n in dims)]
    while int(np.prod(chain[-1])) > coarse_target and all(n % 2 == 0 for n in chain[-1] if n > 1):
        chain.append(tuple(n // 2 if n > 1 else 1 for n in chain[-1]))
    return chain


# --------------------------------------------------------------------------- geometry
def level_scales(chain):
    """Axis scales of every level (the rule of otm_api.cu build: norm*vol/h_a^2)."""
    h = [1.0, 1.0, 1.0]
    norm = 1.0
    out = []
    for li, d in enumerate(chain):
        vol = h[0] * h[1] * h[2]
        out.append(tuple(norm * vol / (h[a] * h[a]) for a in range(3)))
        if li + 1 < len(chain):
            for a in range(3):
                if chain[li + 1][a] < d[a]:
                    h[a] *= 2.0
                    norm *= 0.5
    return out


@dataclass(frozen=True)
class SlabLayout:
    dims: tuple            # global level-0 dims
    world: int
    chain: tuple           # level dims
    scales: tuple          # level axis scales
    nlev_dist: int         # levels 0 .. nlev_dist-1 are distributed; level nlev_dist is agglomerated

    @staticmethod
    def make(dims, world, coarse_target=64, min_local=65536):
        """Levels stay distributed while they split into even slabs of >= 2 planes and
        each rank keeps >= min_local vertices (level 0 always); below that the level
        is agglomerated: the single-GPU V-cycle tail (per-level kernels, single-launch
        bottom) runs it, where a slab level would cost more in launches and halos than
        its work (measured: 2.1x the single-GPU time per PCG iteration at 256^3 on one
        GPU with every level on slabs)."""
        chain = tuple(level_dims(dims, coarse_target))
        nl = len(chain)
        la = 0
        while la < nl - 1:
            nx = chain[la][0]
            nxl = nx // world
            if nx % world or nxl < 2 or nxl % 2 or any(n % 2 for n in chain[la]):
                break
            if any(chain[la + 1][a] * 2 != chain[la][a] for a in range(3)):
                break                               # slab levels need 3-D coarsening
            if la > 0 and int(np.prod(chain[la])) // world < min_local:
                break
            la += 1
        if la == 0:
            raise ValueError(f"dims {tuple(dims)} cannot be split into {world} even slabs of >= 2 planes")
        sc = level_scales(chain)
        if len(set(sc[la])) != 1:
            raise ValueError("the agglomerated level needs equal axis scales")
        return SlabLayout(tuple(dims), world, chain, tuple(sc), la)

    def nxl(self, level):
        return self.chain[level][0] // self.world


# --------------------------------------------------------------------------- comms
def _halo_kernel(dsts, lefts, rights) -> bool:
    """Ghost planes of CUDA slab fields in one launch each (otm_slab_halo_local);
    False when the fields are not contiguous CUDA tensors (the caller copies)."""
    if not all(getattr(t, "is_cuda", False) and t.is_contiguous() for t in (*dsts, *lefts, *rights)):
        return False
    import torch
    from . import _lib
    lib = _lib.load()
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for t, left, right in zip(dsts, lefts, rights):
        ncases = t.shape[0] if t.dim() == 4 else 1
        pl = t.shape[-1] * t.shape[-2]
        rc = lib.otm_slab_halo_local(stream, t.element_size(), ncases, pl, C.c_void_p(t.data_ptr()), t.shape[-3] - 2,
                                     C.c_void_p(left.data_ptr()), left.shape[-3] - 2, C.c_void_p(right.data_ptr()),
                                     right.shape[-3] - 2)
        if rc != 0:
            raise RuntimeError(f"otm_slab_halo_local failed ({rc})")
    return True


class LocalComm:
    """All slabs live in this process (list index = rank); exchanges are copies."""

    def __init__(self, world):
        self.world = world
        self.ranks = list(range(world))

    def halo(self, ts):
        # ghost planes are written, interior planes read: no aliasing, no staging copies
        W = len(ts)
        if _halo_kernel(ts, [ts[(i - 1) % W] for i in range(W)], [ts[(i + 1) % W] for i in range(W)]):
            return
        for i, t in enumerate(ts):
            left, right = ts[(i - 1) % W], ts[(i + 1) % W]
            t.select(-3, 0).copy_(left.select(-3, left.shape[-3] - 2))
            t.select(-3, t.shape[-3] - 1).copy_(right.select(-3, 1))

    def halo_start(self, ts):
        """In-process ghost planes are plain device copies: done at once."""
        self.halo(ts)

    def halo_finish(self, pending):
        pass

    def allreduce(self, vals):
        out = np.zeros_like(np.asarray(vals[0], dtype=np.float64))
        for v in vals:                      # rank order: deterministic
            out = out + np.asarray(v, dtype=np.float64)
        return out

    def gather(self, ts):
        import torch
        return torch.cat([t.narrow(-3, 1, t.shape[-3] - 2) for t in ts], dim=-3)

    def allreduce_dev(self, vals):
        """Sum of per-slab partial sums where they live (device tensors stay on the
        device: no host round trip), in rank order."""
        out = vals[0] + 0
        for v in vals[1:]:
            out = out + v
        return out


class DistComm:
    """One slab per process over torch.distributed (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]

    def halo(self, ts):
        self.halo_finish(self.halo_start(ts))

    def halo_start(self, ts):
        """Post the exchange of the two boundary planes with the neighbours (NCCL runs
        it on its own stream, after the work already queued on the current one) and
        return without waiting: the caller can queue work that does not read the ghost
        planes before halo_finish."""
        (t,) = ts
        dist = self.dist
        r, W = self.ranks[0], self.world
        if W == 1:
            if not _halo_kernel([t], [t], [t]):
                t.select(-3, 0).copy_(t.select(-3, t.shape[-3] - 2))
                t.select(-3, t.shape[-3] - 1).copy_(t.select(-3, 1))
            return None
        last = t.select(-3, t.shape[-3] - 2).contiguous()
        first = t.select(-3, 1).contiguous()
        from_left = last.new_empty(last.shape)
        from_right = first.new_empty(first.shape)
        ops = [dist.P2POp(dist.isend, last, (r + 1) % W, self.group),
               dist.P2POp(dist.isend, first, (r - 1) % W, self.group),
               dist.P2POp(dist.irecv, from_left, (r - 1) % W, self.group),
               dist.P2POp(dist.irecv, from_right, (r + 1) % W, self.group)]
        return dist.batch_isend_irecv(ops), t, from_left, from_right, (last, first)

    def halo_finish(self, pending):
        """Wait for a halo_start exchange (the current stream waits on NCCL's) and
        write the received planes into the ghost planes."""
        if pending is None:
            return
        reqs, t, from_left, from_right, _sent = pending
        for q in reqs:
            q.wait()
        t.select(-3, 0).copy_(from_left)
        t.select(-3, t.shape[-3] - 1).copy_(from_right)

    def allreduce(self, vals):
        import torch
        (v,) = vals
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        tt = torch.tensor(np.asarray(v, dtype=np.float64), device=dev)
        if self.world > 1:
            self.dist.all_reduce(tt, op=self.dist.ReduceOp.SUM, group=self.group)
        return tt.cpu().numpy()

    def allreduce_dev(self, vals):
        """In-place all-reduce of this rank's partial sums: a CUDA tensor is reduced by
        NCCL on the current stream (no host round trip); numpy goes through gloo."""
        import torch
        (v,) = vals
        if isinstance(v, torch.Tensor):
            if self.world > 1:
                self.dist.all_reduce(v, op=self.dist.ReduceOp.SUM, group=self.group)
            return v
        t = torch.from_numpy(np.array(v, dtype=np.float64))
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t.numpy()

    def gather(self, ts):
        import torch
        (t,) = ts
        inner = t.narrow(-3, 1, t.shape[-3] - 2).contiguous()
        if self.world == 1:
            return inner
        parts = [torch.empty_like(inner) for _ in range(self.world)]
        self.dist.all_gather(parts, inner, group=self.group)
        return torch.cat(parts, dim=-3)


# --------------------------------------------------------------------------- CUDA backend
class CudaSlabBackend:
    """The slab kernels of libotm.so (include/otm_slab.h) on torch-allocated device memory."""

    def __init__(self, max_items):
        from . import _dev, _lib
        _dev.require_cuda()
        self.t = _dev.torch()
        self.lib = _lib.load()
        self.ws = self.lib.otm_slab_create(int(max_items))
        if not self.ws:
            raise RuntimeError("otm_slab_create failed")
        self.device = "cuda"
        self.f32 = self.t.float32
        self.f64 = self.t.float64

    def __del__(self):
        try:
            self.lib.otm_slab_destroy(self.ws)
        except Exception:
            pass

    def zeros(self, shape, dtype):
        return self.t.zeros(shape, dtype=dtype, device="cuda")

    def _rc(self, rc):
        if rc != 0:
            msg = self.lib.otm_slab_last_error(self.ws).decode()
            raise (ValueError if rc == 1 else RuntimeError)(f"slab kernel failed ({rc}): {msg}")

    def _sync_stream(self):
        self.lib.otm_slab_set_stream(self.ws, C.c_void_p(self.t.cuda.current_stream().cuda_stream))

    @staticmethod
    def _d3(v):
        return (C.c_double * 3)(*[float(x) for x in v])

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr()) if t is not None else None

    def stencil(self, op, dims, scale, kap, a, f, dinv, omega, o1, o2=None, want_dots=False):
        self._sync_stream()
        out = (C.c_double * 3)()
        self._rc(self.lib.otm_slab_stencil(self.ws, op, *dims, self._d3(scale), self._p(kap), self._p(a),
                                           self._p(f), self._p(dinv), float(omega), self._p(o1), self._p(o2),
                                           out if want_dots else None))
        return np.array(out[:]) if want_dots else None

    # ---- device scalars (otm_slab_set_scalar_mode 1): PCG dots, beta, alpha stay on the device
    def scalars(self, n):
        return self.t.zeros(n, dtype=self.f64, device="cuda")

    @staticmethod
    def to_host(S):
        return S.cpu().numpy()

    @staticmethod
    def put(S, i, v):
        S[i:i + len(v)].copy_(v)

    def pcg_step(self, stage, S):
        self._sync_stream()
        self._rc(self.lib.otm_slab_pcg_step(self.ws, int(stage), self._p(S)))

    def _dev_call(self, fn, *args):
        self.lib.otm_slab_set_scalar_mode(self.ws, 1)
        try:
            return fn(*args)
        finally:
            self.lib.otm_slab_set_scalar_mode(self.ws, 0)

    def stencil_dev(self, op, dims, scale, kap, a, f, dinv, omega, o1, o2=None):
        self._sync_stream()
        out = self.t.empty(3, dtype=self.f64, device="cuda")
        self._rc(self._dev_call(self.lib.otm_slab_stencil, self.ws, op, *dims, self._d3(scale), self._p(kap),
                                self._p(a), self._p(f), self._p(dinv), float(omega), self._p(o1), self._p(o2),
                                C.cast(C.c_void_p(out.data_ptr()), C.POINTER(C.c_double))))
        return out

    def stencil_range(self, op, dims, scale, kap, a, f, dinv, omega, o1, o2, x_lo, x_hi, want_dots=False):
        """otm_slab_stencil_range: only the output planes [x_lo, x_hi) of the ghosted
        slab; want_dots returns the range's dot products as a (3,) device tensor."""
        self._sync_stream()
        if not want_dots:
            self._rc(self.lib.otm_slab_stencil_range(self.ws, op, *dims, self._d3(scale), self._p(kap), self._p(a),
                                                     self._p(f), self._p(dinv), float(omega), self._p(o1),
                                                     self._p(o2), int(x_lo), int(x_hi), None))
            return None
        out = self.t.empty(3, dtype=self.f64, device="cuda")
        self._rc(self._dev_call(self.lib.otm_slab_stencil_range, self.ws, op, *dims, self._d3(scale), self._p(kap),
                                self._p(a), self._p(f), self._p(dinv), float(omega), self._p(o1), self._p(o2),
                                int(x_lo), int(x_hi), C.cast(C.c_void_p(out.data_ptr()), C.POINTER(C.c_double))))
        return out

    def pupd_dev(self, dims, z, p, beta):
        self._sync_stream()
        self._rc(self._dev_call(self.lib.otm_slab_pupd, self.ws, *dims, self._p(z), self._p(p),
                                C.cast(C.c_void_p(beta.data_ptr()), C.POINTER(C.c_double))))

    def upd_dev(self, dims, d, r, p, q, alpha):
        self._sync_stream()
        out = self.t.empty(3, dtype=self.f64, device="cuda")
        self._rc(self._dev_call(self.lib.otm_slab_upd, self.ws, *dims, self._p(d), self._p(r), self._p(p), self._p(q),
                                C.cast(C.c_void_p(alpha.data_ptr()), C.POINTER(C.c_double)),
                                C.cast(C.c_void_p(out.data_ptr()), C.POINTER(C.c_double))))
        return out

    def restrict(self, dims_f, res_f, f_c):
        self._sync_stream()
        self._rc(self.lib.otm_slab_restrict(self.ws, *dims_f, self._p(res_f), self._p(f_c)))

    def prolong(self, dims_f, z_c, z_f):
        self._sync_stream()
        self._rc(self.lib.otm_slab_prolong(self.ws, *dims_f, self._p(z_c), self._p(z_f)))

    def coarsen(self, dims_f, k_f, k_c):
        self._sync_stream()
        self._rc(self.lib.otm_slab_coarsen(self.ws, *dims_f, self._p(k_f), self._p(k_c)))

    def dinv(self, dims, scale, kap, out):
        self._sync_stream()
        self._rc(self.lib.otm_slab_dinv(self.ws, *dims, self._d3(scale), self._p(kap), self._p(out)))

    def pupd(self, dims, z, p, beta):
        self._sync_stream()
        self._rc(self.lib.otm_slab_pupd(self.ws, *dims, self._p(z), self._p(p), self._d3(beta)))

    def upd(self, dims, d, r, p, q, alpha):
        self._sync_stream()
        out = (C.c_double * 3)()
        self._rc(self.lib.otm_slab_upd(self.ws, *dims, self._p(d), self._p(r), self._p(p), self._p(q),
                                       self._d3(alpha), out))
        return np.array(out[:])

    def load_sums(self, dims, scale, kap64):
        self._sync_stream()
        out = (C.c_double * 3)()
        self._rc(self.lib.otm_slab_load_sums(self.ws, *dims, self._d3(scale), self._p(kap64), out))
        return np.array(out[:])

    def res64(self, dims, scale, kap64, T, fmean, r32):
        self._sync_stream()
        out = (C.c_double * 9)()
        self._rc(self.lib.otm_slab_res64(self.ws, *dims, self._d3(scale), self._p(kap64), self._p(T),
                                         self._d3(fmean), self._p(r32), out))
        return np.array(out[:])

    def tupd(self, dims, T, d, mean):
        self._sync_stream()
        self._rc(self.lib.otm_slab_tupd(self.ws, *dims, self._p(T), self._p(d), self._d3(mean)))

    def tensor_sums(self, dims, scale, T, kap64):
        self._sync_stream()
        out = (C.c_double * 6)()
        self._rc(self.lib.otm_slab_tensor_sums(self.ws, *dims, self._d3(scale), self._p(T), self._p(kap64), out))
        return np.array(out[:])

    def filter(self, mode, dims, radius, material, inp, out, kap64=None):
        self._sync_stream()
        sums = (C.c_double * 3)()
        self._rc(self.lib.otm_slab_filter(self.ws, mode, *dims, float(radius), float(material[0]),
                                          float(material[1]), float(material[2]), self._p(inp), self._p(out),
                                          self._p(kap64), sums if mode == 2 else None))
        return np.array(sums[:]) if mode == 2 else None

    def sensitivity(self, dims, n_total, material, T, rho_f, dG, sens_f):
        self._sync_stream()
        self._rc(self.lib.otm_slab_sensitivity(self.ws, *dims, float(n_total), float(material[0]),
                                               float(material[1]), float(material[2]), self._p(T),
                                               self._p(rho_f), (C.c_double * 6)(*[float(v) for v in dG]),
                                               self._p(sens_f)))

    def oc_sums(self, dims, n_total, oc, rho, sens, lams):
        self._sync_stream()
        out = (C.c_double * 32)()
        self._rc(self.lib.otm_slab_oc_sums(self.ws, *dims, float(n_total), C.byref(oc), self._p(rho), self._p(sens),
                                           len(lams), (C.c_double * len(lams))(*lams), out))
        return np.array(out[:len(lams)])

    def oc_apply(self, dims, n_total, oc, rho, sens, lam, rho_out):
        self._sync_stream()
        ch = C.c_double()
        self._rc(self.lib.otm_slab_oc_apply(self.ws, *dims, float(n_total), C.byref(oc), self._p(rho),
                                            self._p(sens), float(lam), self._p(rho_out), C.byref(ch)))
        return ch.value

    # agglomerated coarse levels: the single-GPU hierarchy of that level
    def coarse_hierarchy(self, dims):
        from ._dev import Context
        return Context(dims, jacobi_omega=1.25)     # its top level is a coarse level of the slab problem

    def coarse_build(self, ctx, kap_full32):
        k64 = kap_full32.to(self.f64).contiguous()
        ctx.call("otm_build_kappa", C.c_void_p(k64.data_ptr()))

    def coarse_vcycle(self, ctx, f_full, z_full):
        ctx.call("otm_vcycle", C.c_void_p(f_full.data_ptr()), C.c_void_p(z_full.data_ptr()))


# --------------------------------------------------------------------------- solver
class _Lev:
    pass


class SlabSolver:
    """Distributed solve_cases + effective tensor on x-slabs (homogenize.py:71-122)."""

    def __init__(self, dims, comm, backend, kappa0=1.0, kappa_min=1e-4, penalty=3.0, omega=0.95,
                 omega_coarse=1.25, inner_reduction=1e-5, max_inner=40, tolf=0.85):
        self.L = SlabLayout.make(dims, comm.world)
        self.comm, self.B = comm, backend
        self.kappa0, self.kappa_min, self.penalty = kappa0, kappa_min, penalty
        # the single-GPU solver's knobs (otm_api.cu): Jacobi 0.95 on level 0, 1.25 below,
        # inner PCG target max(1e-5 ||r||, 0.85 tol ||f||)
        self.omega, self.omega_coarse = omega, omega_coarse
        self.inner_reduction, self.max_inner, self.tolf = inner_reduction, max_inner, tolf
        self.ranks = list(comm.ranks)
        B, L = backend, self.L
        f32, f64 = B.f32, B.f64
        self.slabs = []
        for r in self.ranks:
            s = _Lev()
            s.rank = r
            s.levels = []
            for l in range(L.nlev_dist):
                nx, ny, nz = L.chain[l]
                nxl = nx // L.world
                lv = _Lev()
                lv.dims = (nxl, ny, nz)
                lv.kap = B.zeros((nxl + 2, ny, nz), f32)
                lv.dinv = B.zeros((nxl + 2, ny, nz), f32)
                lv.f = B.zeros((3, nxl + 2, ny, nz), f32)
                lv.z = B.zeros((3, nxl + 2, ny, nz), f32)
                lv.res = B.zeros((3, nxl + 2, ny, nz), f32)
                s.levels.append(lv)
            nxl, ny, nz = s.levels[0].dims
            s.kap64 = B.zeros((nxl + 2, ny, nz), f64)
            s.T = B.zeros((3, nxl + 2, ny, nz), f64)
            s.p = B.zeros((3, nxl + 2, ny, nz), f32)
            s.q = B.zeros((3, nxl + 2, ny, nz), f32)
            s.d = B.zeros((3, nxl + 2, ny, nz), f32)
            # the agglomerated level's slab (with ghosts) for the coarse correction
            cx, cy, cz = L.chain[L.nlev_dist]
            cl = cx // L.world
            s.cres = B.zeros((3, cl + 2, cy, cz), f32)
            s.cf = B.zeros((3, cl + 2, cy, cz), f32)
            s.ckap = B.zeros((cl + 2, cy, cz), f32)
            self.slabs.append(s)
        self.coarse = B.coarse_hierarchy(L.chain[L.nlev_dist])
        self.coarse_scale = L.scales[L.nlev_dist][0]
        self.n_total = int(np.prod(dims))
        self.warm = False
        self.fmean = np.zeros(3)
        # halo / stencil overlap: on where the exchange is a real transfer (NCCL between
        # processes); OTM_SLAB_OVERLAP=1 forces it (tests: the split on any comm), =0 off
        import os
        ov = os.environ.get("OTM_SLAB_OVERLAP")
        self.overlap = (ov == "1") if ov is not None else (isinstance(comm, DistComm) and comm.world > 1)

    # ---- helpers
    def _cidx(self, s, device):
        """Planes of the agglomerated level (with ghosts) that slab s keeps, as an index
        tensor on the field's device (built once)."""
        idx = getattr(s, "cidx", None)
        if idx is None:
            import torch
            cl, nxc = self.L.nxl(self.L.nlev_dist), self.L.chain[self.L.nlev_dist][0]
            lo = s.rank * cl
            idx = torch.tensor([(lo - 1 + i) % nxc for i in range(cl + 2)], dtype=torch.long, device=device)
            s.cidx = idx
        return idx

    def _halo(self, get):
        self.comm.halo([get(s) for s in self.slabs])

    def _stencil_after_halo(self, get, level, full, part):
        """The halo exchange of get(s) followed by a stencil reading it: full(s) runs
        the stencil on the whole slab once the ghost planes are in (-> dots or None).
        With self.overlap the stencil is split (SURVEY 8(e) overlap): part(s, lo, hi)
        on the output planes [2, nxl) -- which read no ghost plane -- is queued while
        the exchange is in flight, planes 1 and nxl after it; the three partial dot
        products are added (a different summation order than full())."""
        if not self.overlap:
            self._halo(get)
            return [full(s) for s in self.slabs]
        pending = self.comm.halo_start([get(s) for s in self.slabs])
        n = self.slabs[0].levels[level].dims[0]
        inner = [part(s, 2, n) if n > 2 else None for s in self.slabs]
        self.comm.halo_finish(pending)
        out = []
        for s, di in zip(self.slabs, inner):
            parts = [di, part(s, 1, 2)] + ([part(s, n, n + 1)] if n > 1 else [])
            parts = [d for d in parts if d is not None]
            tot = None
            for d in parts:
                tot = d if tot is None else tot + d
            out.append(tot)
        return out

    def _sum(self, vals):
        return self.comm.allreduce(vals)

    def x0(self, s, level=0):
        return s.rank * self.L.nxl(level)

    # ---- build (solver.py:269-305 on slabs)
    def build_kappa(self, kap64_interiors):
        """kap64_interiors: one (nxl, ny, nz) fp64 device array per local slab (level-0 element factors)."""
        B, L = self.B, self.L
        for s, k in zip(self.slabs, kap64_interiors):
            s.kap64.narrow(0, 1, s.kap64.shape[0] - 2).copy_(k)
        self._halo(lambda s: s.kap64)
        for s in self.slabs:
            s.levels[0].kap.copy_(s.kap64.to(B.f32))
        for l in range(L.nlev_dist):
            if l > 0:
                for s in self.slabs:
                    B.coarsen(s.levels[l - 1].dims, s.levels[l - 1].kap, s.levels[l].kap)
                self._halo(lambda s, l=l: s.levels[l].kap)
            for s in self.slabs:
                lv = s.levels[l]
                B.dinv(lv.dims, L.scales[l], lv.kap, lv.dinv)
            self._halo(lambda s, l=l: s.levels[l].dinv)
        for s in self.slabs:
            top = s.levels[-1]
            B.coarsen(top.dims, top.kap, s.ckap)
        full = self.comm.gather([s.ckap for s in self.slabs])
        B.coarse_build(self.coarse, full.contiguous())

    def build_density(self, rho_f_interiors):
        """SIMP (element.py:91-94) on each slab's interior filtered density, then build."""
        k = [self.kappa_min + (self.kappa0 - self.kappa_min) * r ** self.penalty for r in rho_f_interiors]
        self.build_kappa(k)

    # ---- V-cycle on slabs (solver.py:206-215 with the damped-Jacobi smoother)
    def _vcycle(self):
        B, L = self.B, self.L
        nd = L.nlev_dist
        dots = [None] * len(self.slabs)
        for l in range(nd):
            om = self.omega if l == 0 else self.omega_coarse

            def sm_full(s, l=l, om=om):
                lv = s.levels[l]
                B.stencil(0, lv.dims, L.scales[l], lv.kap, None, lv.f, lv.dinv, om, lv.z, lv.res)

            def sm_part(s, lo, hi, l=l, om=om):
                lv = s.levels[l]
                B.stencil_range(0, lv.dims, L.scales[l], lv.kap, None, lv.f, lv.dinv, om, lv.z, lv.res, lo, hi)

            self._stencil_after_halo(lambda s, l=l: s.levels[l].f, l, sm_full, sm_part)
            self._halo(lambda s, l=l: s.levels[l].res)
            for s in self.slabs:
                lv = s.levels[l]
                dst = s.levels[l + 1].f if l + 1 < nd else s.cf
                B.restrict(lv.dims, lv.res, dst)
        # agglomerated levels: every rank runs the coarse V-cycle on the gathered right-hand side
        f_full = self.comm.gather([s.cf for s in self.slabs]).contiguous()
        z_full = B.zeros(tuple(f_full.shape), B.f32)
        B.coarse_vcycle(self.coarse, f_full, z_full)
        z_full.mul_(1.0 / self.coarse_scale)              # that hierarchy's level 0 carries scale 1
        for s in self.slabs:
            s.cres.copy_(z_full.index_select(1, self._cidx(s, z_full.device)))
        for l in range(nd - 1, -1, -1):
            for s in self.slabs:
                lv = s.levels[l]
                src = s.levels[l + 1].res if l + 1 < nd else s.cres
                B.prolong(lv.dims, src, lv.z)
            om = self.omega if l == 0 else self.omega_coarse

            def jac_full(s, l=l, om=om):
                lv = s.levels[l]
                if l == 0:
                    return B.stencil_dev(1, lv.dims, L.scales[l], lv.kap, lv.z, lv.f, lv.dinv, om, lv.res)
                B.stencil(1, lv.dims, L.scales[l], lv.kap, lv.z, lv.f, lv.dinv, om, lv.res, None)

            def jac_part(s, lo, hi, l=l, om=om):
                lv = s.levels[l]
                return B.stencil_range(1, lv.dims, L.scales[l], lv.kap, lv.z, lv.f, lv.dinv, om, lv.res, None,
                                       lo, hi, want_dots=(l == 0))

            got = self._stencil_after_halo(lambda s, l=l: s.levels[l].z, l, jac_full, jac_part)
            if l == 0:
                dots = got
            if l > 0:
                self._halo(lambda s, l=l: s.levels[l].res)
        return self._pcg_dots(dots)                       # r . z per case (device)

    # ---- solve (solver.py:366-406 semantics, fp64 defect correction)
    def _pcg_dots(self, vals):
        """All-reduced partial sums, left where they live (device for the CUDA backend)."""
        return self.comm.allreduce_dev(vals)

    def solve(self, tol=1e-6, max_vcycles=200, check_every=4):
        """The batched MG-PCG with the PCG scalars on the device: dots are all-reduced in
        device memory and the recurrences run in a one-thread kernel
        (otm_slab_pcg_step), so an inner iteration has no host round trip.  The host
        reads the active flags every `check_every` iterations, and after every
        iteration from two before the previous solve's count on (iterations after a
        case converged apply alpha = 0 to it: no effect on the result, but a whole
        iteration of work -- at 256^3 one iteration costs ~1 ms, a flag read ~30 us).
        Every load case has its own budget of `max_vcycles` preconditioner
        applications (homogenize.py:85-90)."""
        B, L = self.B, self.L
        d0 = self.slabs[0].levels[0].dims
        sc0 = L.scales[0]
        self.fmean = self._sum([B.load_sums(d0, sc0, s.kap64) for s in self.slabs]) / self.n_total
        if not self.warm:
            for s in self.slabs:
                s.T.zero_()
        ccyc = np.zeros(3)

        def residual():
            self._halo(lambda s: s.T)
            sums = self._sum([B.res64(d0, sc0, s.kap64, s.T, self.fmean, s.levels[0].f) for s in self.slabs])
            rr, ff = sums[0:3], sums[3:6]
            fn = np.sqrt(ff)
            rel = np.where(fn > 0, np.sqrt(rr) / np.where(fn > 0, fn, 1.0), 0.0)
            self._sumT = sums[6:9]
            return rel, fn, np.sqrt(rr)

        rel, fn, rn = residual()
        done = (fn == 0) | (rel <= tol)
        if getattr(self, "_S", None) is None:
            self._S = B.scalars(28)
        S = self._S

        def one_iteration():
            rz = self._vcycle()
            B.put(S, 0, rz)
            B.pcg_step(0, S)
            for s in self.slabs:
                B.pupd_dev(d0, s.levels[0].res, s.p, S[6:9])
            pq = self._pcg_dots(self._stencil_after_halo(
                lambda s: s.p, 0,
                lambda s: B.stencil_dev(2, d0, sc0, s.levels[0].kap, s.p, None, None, 0.0, s.q),
                lambda s, lo, hi: B.stencil_range(2, d0, sc0, s.levels[0].kap, s.p, None, None, 0.0, s.q, None,
                                                  lo, hi, want_dots=True)))
            B.put(S, 9, pq)
            B.pcg_step(1, S)
            rr = self._pcg_dots([B.upd_dev(d0, s.d, s.levels[0].f, s.p, s.q, S[12:15]) for s in self.slabs])
            B.put(S, 15, rr)
            B.pcg_step(2, S)

        first_loop = True
        while not done.all():
            pred = self._inner_pred if first_loop else 1
            if ((~done) & (ccyc >= max_vcycles)).any():
                from ._dev import ConvergenceError
                raise ConvergenceError(f"slab solve did not converge in {max_vcycles} V-cycles per case",
                                       float(rel.max()))
            init = np.zeros(28)
            init[18:21] = np.maximum(self.inner_reduction * rn, self.tolf * tol * fn) ** 2
            init[21:24] = (~done).astype(np.float64)
            init[24] = 1.0
            init[25:28] = ccyc
            B.put(S, 0, init if not hasattr(S, "copy_") else B.t.from_numpy(init).to(S.device))
            for s in self.slabs:
                s.d.zero_()
                s.p.zero_()
            for it in range(self.max_inner):
                g = self._pcg_graph
                if g is not None:
                    g.replay()
                else:
                    one_iteration()
                    if self._graph_ok and it == 0:
                        self._capture(one_iteration)
                if (it + 1) % check_every == 0 or it + 1 >= pred - 2 or it + 1 == self.max_inner:
                    h = B.to_host(S)
                    active = h[21:24] != 0
                    if not active.any() or (active & (h[25:28] >= max_vcycles)).any():
                        break
            if first_loop:
                self._inner_pred = it + 1
                first_loop = False
            h = B.to_host(S)
            ccyc = h[25:28].copy()
            for s in self.slabs:
                B.tupd(d0, s.T, s.d, np.zeros(3))
            rel, fn, rn = residual()
            done = (fn == 0) | (rel <= tol)
        # mean projection of the solution (solver.py:404-406); sum T from the last defect pass
        mean = self._sumT / self.n_total
        for s in self.slabs:
            B.tupd(d0, s.T, None, mean)
        self.warm = True
        self.cycles = int(ccyc.sum())
        return self.cycles

    # one inner PCG iteration as a CUDA graph (the per-call host overhead of the slab
    # orchestration -- ~60 small launches per iteration issued from Python -- exceeded
    # the GPU time at 256^3); in-process slabs only, unless OTM_SLAB_GRAPH=1 (NCCL
    # collectives inside a captured graph are untested on this single-GPU project)
    _pcg_graph = None
    _inner_pred = 1          # inner iterations of the previous solve's first loop

    @property
    def _graph_ok(self):
        import os
        if getattr(self, "_graph_failed", False) or not hasattr(self.B, "pcg_step") or self.B.device != "cuda":
            return False
        if isinstance(self.comm, LocalComm):
            return os.environ.get("OTM_SLAB_GRAPH", "1") != "0"
        return os.environ.get("OTM_SLAB_GRAPH") == "1"

    def _capture(self, fn):
        import torch
        try:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            torch.cuda.synchronize()
            self._pcg_graph = g
        except Exception:                     # stay on the eager loop for this solver
            self._graph_failed = True
            self._pcg_graph = None
            torch.cuda.synchronize()

    def tensor(self):
        """kappa_H (homogenize.py:103-122): all-reduced element-energy sums / N."""
        B, L = self.B, self.L
        d0 = self.slabs[0].levels[0].dims
        self._halo(lambda s: s.T)
        sums = self._sum([B.tensor_sums(d0, L.scales[0], s.T, s.kap64) for s in self.slabs])
        return sums / self.n_total

    def fields(self):
        """The full 3-case temperature fields (gathered; for tests)."""
        return self.comm.gather([s.T for s in self.slabs])


# --------------------------------------------------------------------------- design loop
class SlabDesignRun:
    """run_optimization (optimize.py:257-379, model 'oc' with the adaptive-volume
    governor) on x-slabs: every field is a ghosted slab, every scalar all-reduced,
    and the host-side logic (objective, governor, OC multiplier search, convergence
    rule) replayed identically on every rank from identical sums."""

    def __init__(self, config, comm, backend, rho_interiors):
        from . import _lib
        from .optimize import KIND_CODE, Model, _check_supported
        _check_supported(config)
        if config.model is not Model.ADAPTIVE_OC:
            raise NotImplementedError("the slab design loop runs the reference default model 'oc'")
        if config.symmetry == "central":
            raise NotImplementedError("central symmetry mirrors across slabs; not supported on the slab path")
        if not (1.0 <= config.filter.radius <= 2.0):
            raise NotImplementedError("the slab filter needs radius <= 2 (one ghost plane)")
        self.cfg = config
        self.comm, self.B = comm, backend
        mp = config.material
        self.material = (mp.kappa0, mp.kappa_min, mp.penalty)
        # one solver (slab buffers, captured PCG graph) per grid and transport, reused by
        # later runs; every run starts cold
        cache = backend.__dict__.setdefault("_solvers", {})
        key = (tuple(config.dims), comm.world, tuple(comm.ranks), mp.kappa0, mp.kappa_min, mp.penalty, id(comm))
        self.solver = cache.get(key)
        if self.solver is None:
            cache.clear()
            self.solver = SlabSolver(config.dims, comm, backend, kappa0=mp.kappa0, kappa_min=mp.kappa_min,
                                     penalty=mp.penalty)
            cache[key] = self.solver
        self.solver.warm = False
        self.n = self.solver.n_total
        self.lib = _lib.load()
        self.cc = _lib.RunConfigC()
        from .optimize import _run_config_c
        self.cc = _run_config_c(config)
        self.st = _lib.RunStateC()
        self.lib.otm_run_init(C.byref(self.st), C.byref(self.cc))
        self.kind = KIND_CODE[config.target.kind]
        self.oc = config.oc._to_c()
        f64 = backend.f64
        self.parts = []
        for s, r in zip(self.solver.slabs, rho_interiors):
            nxl, ny, nz = s.levels[0].dims
            p = _Lev()
            p.rho = backend.zeros((nxl + 2, ny, nz), f64)
            p.rho.narrow(0, 1, nxl).copy_(r)
            p.rho_f = backend.zeros((nxl + 2, ny, nz), f64)
            p.kap = backend.zeros((nxl + 2, ny, nz), f64)        # ghosted like every slab field
            p.sens_f = backend.zeros((nxl + 2, ny, nz), f64)
            p.sens = backend.zeros((nxl + 2, ny, nz), f64)
            self.parts.append(p)
        self.log = []
        self.kappa = None

    @property
    def finished(self):
        return bool(self.st.finished)

    def _halo(self, get):
        self.comm.halo([get(p) for p in self.parts])

    def _sum(self, vals):
        return self.comm.allreduce(vals)

    def evaluate(self):
        import time
        from .optimize import IterationRecord
        B, cfg, st = self.B, self.cfg, self.st
        t0 = time.perf_counter()
        d0 = self.solver.slabs[0].levels[0].dims
        it = st.iter + 1
        self._halo(lambda p: p.rho)
        sums = self._sum([B.filter(2, d0, cfg.filter.radius, self.material, p.rho, p.rho_f, p.kap)
                          for p in self.parts])
        mean_rho, mean_rho_p, mean_rf = sums / self.n
        self.solver.build_kappa([p.kap.narrow(0, 1, p.kap.shape[0] - 2) for p in self.parts])
        self.solver.solve(tol=cfg.solver_tol, max_vcycles=cfg.max_vcycles)
        kap = self.solver.tensor()
        g = C.c_double()
        dG = (C.c_double * 6)()
        self.lib.otm_objective(self.kind, (C.c_double * 6)(*self.cc.target), (C.c_double * 6)(*kap), C.byref(g), dG)
        g = g.value
        for s, p in zip(self.solver.slabs, self.parts):
            B.sensitivity(d0, self.n, self.material, s.T, p.rho_f, dG[:], p.sens_f)
        self._halo(lambda p: p.sens_f)
        for p in self.parts:
            B.filter(1, d0, cfg.filter.radius, self.material, p.sens_f, p.sens)
        st.iter = it
        # convergence (optimize.py:327-345), as otm_run_step
        if st.have_g_last and abs(g - st.g_last) < cfg.conv_threshold:
            st.plateau += 1
        else:
            st.plateau = 0
        st.g_last = g
        st.have_g_last = 1
        conv = False
        if g <= 1e-12:
            conv = True
        elif st.plateau >= 3:
            cd = st.gov.gap * st.gov.df if st.gov.reduced else float("inf")
            conv = cd < 1e-4 and g <= st.gov.bound
        st.converged = int(conv)
        st.g, st.mean_rho, st.mean_rho_p = g, mean_rho, mean_rho_p
        if conv or it == cfg.max_iter:
            st.finished = 1
        rec = IterationRecord(it, g, mean_rho, mean_rf, st.gov.vstar, self.solver.cycles,
                              (time.perf_counter() - t0) * 1e3)
        self.log.append(rec)
        from .homogenize import ConductivityTensor
        self.kappa = ConductivityTensor(np.array(kap))
        return rec

    # OC multiplier search (optimize.py:114-160): the reference's free step, bracket
    # (l2 *= 4, at most 200 steps) and bisection with its two stopping rules, with the
    # candidate means evaluated 32 at a time (bracket values, or the depth-5 subtree of
    # bisection midpoints) -- the same multipliers the reference visits
    def _means(self, lams):
        d0 = self.solver.slabs[0].levels[0].dims
        return self._sum([self.B.oc_sums(d0, self.n, self.oc, p.rho, p.sens, lams) for p in self.parts]) / self.n

    def _search(self, V):
        tol = self.oc.bisection_tol
        lams = [0.0] + [4.0 ** k for k in range(31)]
        m = self._means(lams)
        if m[0] <= V:
            return 0.0
        l2, it, k0 = 1.0, 0, 1
        while True:
            hit = False
            for k in range(k0, len(lams)):
                if m[k] <= V:
                    hit = True
                    break
                l2 *= 4.0
                it += 1
                if it >= 200:
                    hit = True
                    break
            if hit:
                break
            lams = [l2 * 4.0 ** j for j in range(min(32, 200 - it))]
            m = self._means(lams)
            k0 = 0
        l1 = 1e-30
        while True:
            lo, hi, mids = [l1], [l2], []
            for i in range(31):
                mid = 0.5 * (lo[i] + hi[i])
                mids.append(mid)
                if 2 * i + 2 < 31:
                    lo += [lo[i], mid]
                    hi += [mid, hi[i]]
            m = self._means(mids)
            node = 0
            while True:
                if not ((l2 - l1) / (l1 + l2) > 1e-13):
                    return 0.5 * (l1 + l2)
                if node >= 31:
                    break
                mid = 0.5 * (l1 + l2)
                cur = m[node]
                if cur > V:
                    l1, node = mid, 2 * node + 2
                else:
                    l2, node = mid, 2 * node + 1
                if abs(cur - V) <= tol:
                    return 0.5 * (l1 + l2)

    def _oc_update(self, V):
        d0 = self.solver.slabs[0].levels[0].dims
        lam = self._search(V)
        changed = self._sum([np.array([self.B.oc_apply(d0, self.n, self.oc, p.rho, p.sens, lam, p.rho)])
                             for p in self.parts])
        return changed[0] > 0

    def update(self):
        st, cfg = self.st, self.cfg
        vb = self.lib.otm_governor_update(C.byref(st.gov), st.g, st.mean_rho, st.mean_rho_p)
        vb = min(vb, st.mean_rho + 0.5 * cfg.oc.step_limit)
        if not self._oc_update(vb):
            self._oc_update(st.mean_rho - 0.25 * cfg.oc.step_limit)

    def step(self):
        rec = self.evaluate()
        if not self.finished:
            self.update()
        return rec

    def density(self):
        """The full density field (gathered)."""
        return self.comm.gather([p.rho for p in self.parts])
