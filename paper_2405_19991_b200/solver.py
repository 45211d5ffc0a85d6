"""Periodic conduction operator and its multigrid solver (reference: solver.py).

The B200 hierarchy is a libotm context: the level chain, the element factors per
level and every workspace live on the device.  ``solve_equation`` drives the
batched mixed-precision MG-PCG to the reference's stopping
rule ||f - K T|| / ||f|| <= tol evaluated in fp64.
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _dev
from ._dev import ConvergenceError  # noqa: F401  (re-exported API name)
from .element import MaterialParams, template_matrix


class GridLevel:
    """Read-only view of one level (solver.py:66-83): dims, axis scales, template."""

    def __init__(self, hier, index, dims, axis_scale):
        self._hier = hier
        self.index = index
        self.dims = tuple(dims)
        self.axis_scale = tuple(axis_scale)
        self.template = template_matrix(axis_scale)

    @property
    def num_vertices(self) -> int:
        nx, ny, nz = self.dims
        return nx * ny * nz


class GridHierarchy:
    """Level stack down to a direct solve (solver.py:203-247), device resident.

    ``dtype`` and ``smooth_sweeps`` are accepted for API compatibility: the B200
    solver always meets the fp64 residual contract (fp64 defect correction around
    an fp32 MG-PCG) and smooths with one damped-Jacobi sweep each way."""

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

    def build(self, kappa_elems) -> None:
        """Install element factors and set up every level (solver.py:269-275)."""
        k, _ = _dev.to_device(kappa_elems)
        if tuple(k.shape) != self.dims:
            raise ValueError(f"kappa shape {tuple(k.shape)} != level dims {self.dims}")
        if float(k.min()) <= 0.0:
            raise RuntimeError("non-positive relaxation diagonal; check conductivities")
        self.ctx.call("otm_build_kappa", _dev.ptr(k))
        self.built = True

    def build_density(self, rho_filtered, mp: MaterialParams) -> None:
        """simp_conductivity + build, fused on the device (homogenize.py:84-85)."""
        rf, _ = _dev.to_device(rho_filtered, shape=self.dims)
        self.set_material(mp)
        self.ctx.call("otm_build", _dev.ptr(rf))
        self.built = True

    def _require_built(self):
        if not self.built:
            raise RuntimeError("hierarchy not built; call build() first")

    def solve3(self, f3=None, tol=1e-6, max_vcycles=200, warm=None):
        """Batched solve of three load cases; returns (T (3,nx,ny,nz) tensor, cycles, residuals)."""
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
        rc = ctx.lib.otm_solve(ctx.h, fptr, float(tol), int(max_vcycles), C.byref(cyc), res)
        ctx.version += 1
        self.residual_history = [float(max(res))]
        ctx.check(rc, residual=max(res))
        T = ctx.empty(3, *self.dims)
        ctx.call("otm_get_T", _dev.ptr(T))
        return T, int(cyc.value), [float(r) for r in res]


def apply_K(level: GridLevel, T):
    """Matrix-free K T on the finest level in fp64 (solver.py:111-119)."""
    hier = level._hier
    if level.index != 0:
        raise NotImplementedError("apply_K is exposed for the finest level only")
    hier._require_built()
    t, host = _dev.to_device(T, shape=level.dims)
    out = hier.ctx.empty(*level.dims)
    hier.ctx.call("otm_apply_K", _dev.ptr(t), _dev.ptr(out))
    return _dev.like_input(out, host)


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

    Returns ``(T, cycles)`` with mean(T) = 0; raises ConvergenceError."""
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
    return _dev.like_input(T[0].contiguous(), host), cycles
