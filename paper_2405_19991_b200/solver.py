"""Periodic conduction operator and its multigrid solver (reference: solver.py).

The B200 hierarchy is a libotm context: the level chain, the element factors per
level and every workspace live on the device.  ``solve_equation`` drives the
batched mixed-precision MG-PCG to the reference's stopping
rule ||f - K T|| / ||f|| <= tol evaluated in fp64.

The reference also exposes its V-cycle pieces as functions over mutable level
arrays (``GridLevel.T/f/r``): ``relax_gs8``, ``restrict``, ``prolong_correct``,
``coarse_solve``, ``GridHierarchy.vcycle`` and ``apply_K`` on any level.  Here
the level arrays are host mirrors (numpy, the hierarchy's dtype, created on
first access) and every one of those functions runs on the device in fp64
(``otm_levelops.cu``, reached through ``include/otm.h``): inputs are uploaded
from the mirrors, results written back into them in place, so code written
against the reference (``lev.f[...] = f; relax_gs8(lev)``) behaves the same.
"""

from __future__ import annotations

import ctypes as C
import warnings
from typing import Optional

import numpy as np

from . import _dev
from ._dev import ConvergenceError  # noqa: F401  (re-exported API name)
from .element import MaterialParams, template_matrix

_HIST_CAP = 1 << 16


class GridLevel:
    """One multigrid level (solver.py:66-83): dims, axis scales, template, the
    mutable level arrays ``T``, ``f``, ``r`` and the element factors ``kappa``."""

    def __init__(self, hier, index, dims, axis_scale):
        self._hier = hier
        self.index = index
        self.dims = tuple(dims)
        self.axis_scale = tuple(axis_scale)
        self.template = template_matrix(axis_scale)
        self.dtype = hier.dtype
        self._arrays: dict = {}
        self._kappa = None
        self._kappa_build = -1

    @property
    def num_vertices(self) -> int:
        nx, ny, nz = self.dims
        return nx * ny * nz

    def _array(self, name):
        a = self._arrays.get(name)
        if a is None:
            a = np.zeros(self.dims, dtype=self.dtype)
            self._arrays[name] = a
        return a

    def _assign(self, name, value):
        self._array(name)[...] = value

    T = property(lambda self: self._array("T"), lambda self, v: self._assign("T", v))
    f = property(lambda self: self._array("f"), lambda self, v: self._assign("f", v))
    r = property(lambda self: self._array("r"), lambda self, v: self._assign("r", v))

    @property
    def kappa(self) -> Optional[np.ndarray]:
        """Child-mean element factors of this level (solver.py:257-267); None before build."""
        h = self._hier
        if not h.built:
            return None
        if self._kappa_build != h._build_id:
            k = h.ctx.empty(*self.dims)
            h.ctx.call("otm_level_kappa", int(self.index), _dev.ptr(k))
            self._kappa = k.cpu().numpy().astype(self.dtype, copy=False)
            self._kappa_build = h._build_id
        return self._kappa

    # device copies of the mirrors (fp64) and back
    def _up(self, name):
        return _dev.to_device(self._array(name), shape=self.dims)[0]

    def _down(self, name, t):
        self._array(name)[...] = t.cpu().numpy()


class GridHierarchy:
    """Level stack down to a direct solve (solver.py:203-247), device resident.

    The hot-path solver (``solve_equation``/``solve_cases``) always meets the fp64
    residual contract (fp64 defect correction around an fp32 MG-PCG with a
    damped-Jacobi V-cycle), whatever ``dtype`` says; ``dtype`` is the dtype of the
    level arrays and ``smooth_sweeps`` the Gauss-Seidel sweeps of the API-level
    ``vcycle()``, as in the reference."""

    def __init__(self, dims, dtype=np.float32, smooth_sweeps=(1, 1), coarse_target=64, direct_limit=40000,
                 material: Optional[MaterialParams] = None, filter_radius: float = 1.5, **solver):
        dims = tuple(int(n) for n in dims)
        if len(dims) != 3 or any(n < 1 for n in dims):
            raise ValueError(f"dims must be three positive integers, got {dims}")
        mp = material or MaterialParams()
        self.dtype = np.dtype(dtype)
        self.pre_sweeps, self.post_sweeps = smooth_sweeps
        self.ctx = _dev.Context(dims, kappa0=mp.kappa0, kappa_min=mp.kappa_min, penalty=mp.penalty,
                                radius=filter_radius, coarse_target=coarse_target, direct_limit=direct_limit,
                                **solver)
        self._material = mp
        self.levels = [GridLevel(self, i, d, s) for i, (d, s) in enumerate(self.ctx.levels())]
        self.residual_history: list[float] = []
        self.built = False
        self._build_id = 0

    @property
    def dims(self):
        return self.levels[0].dims

    @property
    def num_levels(self) -> int:
        return len(self.levels)

    def set_material(self, mp: MaterialParams):
        if mp != self._material:
            self.ctx.call("otm_set_material", float(mp.kappa0), float(mp.kappa_min), float(mp.penalty))
            self._material = mp

    def _built_now(self):
        self.built = True
        self._build_id += 1

    def build(self, kappa_elems) -> None:
        """Install element factors and set up every level (solver.py:269-275)."""
        k, _ = _dev.to_device(kappa_elems)
        if tuple(k.shape) != self.dims:
            raise ValueError(f"kappa shape {tuple(k.shape)} != level dims {self.dims}")
        if float(k.min()) <= 0.0:
            raise RuntimeError("non-positive relaxation diagonal; check conductivities")
        self.ctx.call("otm_build_kappa", _dev.ptr(k))
        self._built_now()

    def build_density(self, rho_filtered, mp: MaterialParams) -> None:
        """simp_conductivity + build, fused on the device (homogenize.py:84-85)."""
        rf, _ = _dev.to_device(rho_filtered, shape=self.dims)
        self.set_material(mp)
        self.ctx.call("otm_build", _dev.ptr(rf))
        self._built_now()

    def _require_built(self):
        if not self.built:
            raise RuntimeError("hierarchy not built; call build() first")

    def solve3(self, f3=None, tol=1e-6, max_vcycles=200, warm=None):
        """Batched solve of three load cases; returns (T (3,nx,ny,nz) tensor, cycles, residuals).

        Every case has its own budget of ``max_vcycles`` preconditioner applications
        (homogenize.py:85-90 runs three independent solves); ``cycles`` is their sum."""
        self._require_built()
        ctx = self.ctx
        if warm is not None:
            w, _ = _dev.to_device(warm, shape=(3,) + self.dims)
            ctx.call("otm_set_warm", _dev.ptr(w))
        else:
            ctx.call("otm_set_warm", None)
        fptr = None
        if f3 is not None:
            f3, _ = _dev.to_device(f3, shape=(3,) + self.dims)
            fptr = _dev.ptr(f3)
        cyc = C.c_int(0)
        res = (C.c_double * 3)()
        cur = _dev.torch().cuda.current_stream()
        ctx.stream.wait_stream(cur)
        rc = ctx.lib.otm_solve(ctx.h, fptr, float(tol), int(max_vcycles), C.byref(cyc), res)
        cur.wait_stream(ctx.stream)
        ctx.version += 1
        self.residual_history = self._history()
        ctx.check(rc, residual=max(res))
        T = ctx.empty(3, *self.dims)
        ctx.call("otm_get_T", _dev.ptr(T))
        return T, int(cyc.value), [float(r) for r in res]

    def _history(self):
        buf = (C.c_double * _HIST_CAP)()
        n = self.ctx.lib.otm_residual_history(self.ctx.h, buf, _HIST_CAP)
        return [float(buf[i]) for i in range(min(n, _HIST_CAP))]

    # ---- the reference's V-cycle pieces (solver.py:298-338) -----------------
    def coarse_solve(self) -> None:
        """Direct solve on the coarsest level with the mean pinned to zero (solver.py:307-324)."""
        self._require_built()
        level = self.levels[-1]
        f = level.f.ravel().astype(np.float64)
        total = f.sum()
        scale = np.abs(f).sum()
        if scale > 0 and abs(total) > 1e-4 * scale:
            warnings.warn("coarse load has a nonzero mean component; projecting it out", RuntimeWarning)
        fd = level._up("f")
        T = self.ctx.empty(*level.dims)
        self.ctx.call("otm_coarse_solve", _dev.ptr(fd), _dev.ptr(T))
        level._down("T", T)

    def vcycle(self) -> None:
        """One V-cycle of the reference's multigrid (solver.py:326-338) on the level
        arrays: ``pre_sweeps``/``post_sweeps`` 8-colour Gauss-Seidel sweeps, full
        weighting, the pinned direct solve, trilinear correction -- all on the device
        in fp64, with the level arrays synchronised once before and once after."""
        self._require_built()
        t = _dev.torch()
        ctx = self.ctx
        L = len(self.levels) - 1
        T = [None] * (L + 1)
        F = [None] * (L + 1)
        R = [None] * (L + 1)
        T[0], F[0] = self.levels[0]._up("T"), self.levels[0]._up("f")
        for li in range(L):
            lev = self.levels[li]
            if li > 0:
                T[li] = t.zeros(lev.dims, dtype=t.float64, device="cuda")
            ctx.call("otm_relax_gs8", li, _dev.ptr(T[li]), _dev.ptr(F[li]), int(self.pre_sweeps))
            R[li] = ctx.empty(*lev.dims)
            ctx.call("otm_level_apply", li, _dev.ptr(T[li]), _dev.ptr(F[li]), _dev.ptr(R[li]))
            F[li + 1] = ctx.empty(*self.levels[li + 1].dims)
            ctx.call("otm_restrict", li, _dev.ptr(R[li]), _dev.ptr(F[li + 1]))
        fc = F[L].double()
        total, scale = float(fc.sum()), float(fc.abs().sum())
        if scale > 0 and abs(total) > 1e-4 * scale:
            warnings.warn("coarse load has a nonzero mean component; projecting it out", RuntimeWarning)
        T[L] = ctx.empty(*self.levels[L].dims)
        ctx.call("otm_coarse_solve", _dev.ptr(F[L]), _dev.ptr(T[L]))
        for li in range(L - 1, -1, -1):
            ctx.call("otm_prolong_correct", li, _dev.ptr(T[li]), _dev.ptr(T[li + 1]))
            ctx.call("otm_relax_gs8", li, _dev.ptr(T[li]), _dev.ptr(F[li]), int(self.post_sweeps))
        for li, lev in enumerate(self.levels):
            lev._down("T", T[li])
            lev._down("f", F[li])
            if R[li] is not None:
                lev._down("r", R[li])


def apply_K(level: GridLevel, T):
    """Matrix-free K T on any level in fp64 (solver.py:111-119)."""
    hier = level._hier
    hier._require_built()
    t, host = _dev.to_device(T, shape=level.dims)
    out = hier.ctx.empty(*level.dims)
    if level.index == 0:
        hier.ctx.call("otm_apply_K", _dev.ptr(t), _dev.ptr(out))
    else:
        hier.ctx.call("otm_level_apply", int(level.index), _dev.ptr(t), None, _dev.ptr(out))
    return _dev.like_input(out, host)


def relax_gs8(level: GridLevel, sweeps: int = 1) -> None:
    """Gauss-Seidel by parity colours on ``level.T`` in place (solver.py:131-164),
    one device launch per colour in the reference's colour order."""
    for n in level.dims:
        if n > 1 and n % 2:
            raise ValueError(f"relaxation needs even axes, got dims {level.dims}")
    hier = level._hier
    hier._require_built()
    T, f = level._up("T"), level._up("f")
    hier.ctx.call("otm_relax_gs8", int(level.index), _dev.ptr(T), _dev.ptr(f), int(sweeps))
    level._down("T", T)


def restrict(level_f: GridLevel, level_c: GridLevel) -> None:
    """Full-weighting restriction of ``level_f.r`` into ``level_c.f`` (solver.py:167-177)."""
    if level_c.index != level_f.index + 1:
        raise ValueError("restrict needs consecutive levels (fine, next coarser)")
    hier = level_f._hier
    hier._require_built()
    r = level_f._up("r")
    fc = hier.ctx.empty(*level_c.dims)
    hier.ctx.call("otm_restrict", int(level_f.index), _dev.ptr(r), _dev.ptr(fc))
    level_c._down("f", fc)


def prolong_correct(level_f: GridLevel, level_c: GridLevel) -> None:
    """Trilinear interpolation of ``level_c.T`` added to ``level_f.T`` (solver.py:180-200)."""
    if level_c.index != level_f.index + 1:
        raise ValueError("prolong_correct needs consecutive levels (fine, next coarser)")
    hier = level_f._hier
    hier._require_built()
    Tf, Tc = level_f._up("T"), level_c._up("T")
    hier.ctx.call("otm_prolong_correct", int(level_f.index), _dev.ptr(Tf), _dev.ptr(Tc))
    level_f._down("T", Tf)


def coarse_solve(hier: GridHierarchy) -> np.ndarray:
    """Direct solve of the coarsest level; returns its zero-mean temperature (solver.py:341-344)."""
    hier.coarse_solve()
    return hier.levels[-1].T


def assemble_macro_load(hier: GridHierarchy, case: int, as_tensor: bool = False):
    """Unit-gradient vertex loads (solver.py:347-363)."""
    if case not in (0, 1, 2):
        raise ValueError(f"load case must be 0, 1 or 2, got {case}")
    hier._require_built()
    out = hier.ctx.empty(*hier.dims)
    hier.ctx.call("otm_macro_load", int(case), _dev.ptr(out))
    return out if as_tensor else out.cpu().numpy()


def solve_equation(hier: GridHierarchy, f, tol: float = 1e-6, max_vcycles: int = 200, x0=None):
    """Solve K T = f - mean(f) to ||r|| / ||f|| <= tol (solver.py:366-406).

    Returns ``(T, cycles)`` with mean(T) = 0; raises ConvergenceError.
    ``hier.residual_history`` holds one relative residual per V-cycle."""
    shape = tuple(f.shape)
    if shape != hier.dims:
        raise ValueError(f"load shape {shape} != grid dims {hier.dims}")
    t = _dev.torch()
    fd, host = _dev.to_device(f)
    f3 = t.zeros((3,) + hier.dims, dtype=t.float64, device="cuda")
    f3[0] = fd
    warm = None
    if x0 is not None:
        xd, _ = _dev.to_device(x0, shape=hier.dims)
        warm = t.zeros_like(f3)
        warm[0] = xd
    T, cycles, _ = hier.solve3(f3, tol=tol, max_vcycles=max_vcycles, warm=warm)
    out = _dev.like_input(T[0].contiguous(), host)
    lev = hier.levels[0]
    if "T" in lev._arrays:             # keep materialised level arrays in step (solver.py:388-403)
        lev._down("T", T[0])
    if "f" in lev._arrays:
        lev._down("f", fd - fd.mean())
    return out, cycles
