"""Periodic density fields: seeds, the radial filter, central symmetry
(reference: field.py).

``filter_forward`` / ``filter_backward`` / ``project_central_symmetry`` run on
the device (libotm).  Seed generation (``init_density``) is one-shot host setup
outside the hot loop and stays numpy.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _dev

PATTERN_FLOOR = 0.001          # field.py:18
PATTERN_KINDS = ("p", "d", "g", "iwp", "ball", "random")
_PATTERN_ALIASES = {"p": "p", "d": "d", "g": "g", "iwp": "iwp", "ball": "ball", "centerball": "ball",
                    "random": "random"}


def _check_dims(dims):
    dims = tuple(int(n) for n in dims)
    if len(dims) != 3 or any(n < 1 for n in dims):
        raise ValueError(f"dims must be three positive integers, got {dims}")
    return dims


@dataclass
class DensityField:
    """Design densities and their gradient (field.py:22-50).  ``rho`` / ``grad`` may
    be numpy arrays or CUDA tensors."""

    dims: tuple
    rho: object
    grad: object

    @classmethod
    def zeros(cls, dims) -> "DensityField":
        dims = _check_dims(dims)
        return cls(dims, np.zeros(dims), np.zeros(dims))

    @classmethod
    def from_array(cls, rho) -> "DensityField":
        if hasattr(rho, "data_ptr"):
            if rho.dim() != 3:
                raise ValueError(f"density array must be 3-d, got shape {tuple(rho.shape)}")
            if float(rho.min()) < 0.0 or float(rho.max()) > 1.0:
                raise ValueError("densities must lie in [0, 1]")
            return cls(tuple(rho.shape), rho.clone(), rho.new_zeros(rho.shape))
        rho = np.asarray(rho, dtype=np.float64)
        if rho.ndim != 3:
            raise ValueError(f"density array must be 3-d, got shape {rho.shape}")
        if rho.min() < 0.0 or rho.max() > 1.0:
            raise ValueError("densities must lie in [0, 1]")
        return cls(tuple(rho.shape), rho.copy(), np.zeros(rho.shape))

    @property
    def num_elements(self) -> int:
        nx, ny, nz = self.dims
        return nx * ny * nz

    def mean(self) -> float:
        if hasattr(self.rho, "data_ptr"):
            return float(self.rho.double().mean())
        return float(self.rho.mean(dtype=np.float64))


def cone_kernel(radius: float) -> Callable:
    def kernel(dist):
        return np.maximum(0.0, radius - dist)
    return kernel


@dataclass
class FilterSpec:
    """Cone filter of radius r (field.py:69-93).  Custom ``kernel`` callables are
    not part of the device path and are rejected by the filter entry points."""

    radius: float = 1.5
    kernel: Callable | None = None

    def __post_init__(self):
        if self.radius < 1.0:
            raise ValueError(f"filter radius must be >= 1, got {self.radius}")

    def offsets_and_weights(self):
        kern = self.kernel if self.kernel is not None else cone_kernel(self.radius)
        reach = int(np.ceil(self.radius)) - 1
        span = np.arange(-reach, reach + 1)
        dx, dy, dz = np.meshgrid(span, span, span, indexing="ij")
        dist = np.sqrt(dx ** 2 + dy ** 2 + dz ** 2).ravel()
        w = np.asarray(kern(dist), dtype=np.float64)
        if (w < 0.0).any():
            raise ValueError("filter kernel produced negative weights")
        keep = w > 0.0
        offs = np.stack([dx.ravel(), dy.ravel(), dz.ravel()], axis=1)[keep]
        w = w[keep]
        return offs, w / w.sum()


@dataclass
class InitPattern:
    """Seed geometry (field.py:113-131)."""

    kind: str = "iwp"
    target_volume_fraction: float = 0.5
    seed: int = 0

    def __post_init__(self):
        key = str(self.kind).lower()
        if key not in _PATTERN_ALIASES:
            raise ValueError(f"unknown init pattern {self.kind!r}; choose from {PATTERN_KINDS}")
        self.kind = _PATTERN_ALIASES[key]
        vf = self.target_volume_fraction
        if not (0.0 < vf < 1.0):
            raise ValueError(f"target volume fraction must be in (0, 1), got {vf}")


def _level_set(kind, dims):
    ang = [2.0 * np.pi * (np.arange(n) + 0.5) / n for n in dims]
    X, Y, Z = np.meshgrid(*ang, indexing="ij")
    c, s = (np.cos(X), np.cos(Y), np.cos(Z)), (np.sin(X), np.sin(Y), np.sin(Z))
    if kind == "p":
        return c[0] + c[1] + c[2]
    if kind == "g":
        return s[0] * c[1] + s[1] * c[2] + s[2] * c[0]
    if kind == "d":
        return s[0] * s[1] * s[2] + s[0] * c[1] * c[2] + c[0] * s[1] * c[2] + c[0] * c[1] * s[2]
    return 2.0 * (c[0] * c[1] + c[1] * c[2] + c[2] * c[0]) - (np.cos(2 * X) + np.cos(2 * Y) + np.cos(2 * Z))


def _by_rank(values, vf):
    m = values.size
    k = min(max(int(round(m * (vf - PATTERN_FLOOR) / (1.0 - PATTERN_FLOOR))), 0), m)
    order = np.argsort(values.ravel(), kind="stable")[::-1]
    out = np.full(m, PATTERN_FLOOR)
    out[order[:k]] = 1.0
    return out.reshape(values.shape)


def init_density(dims, pattern: InitPattern) -> DensityField:
    """Periodic seed at the target mean (field.py:192-219); host numpy."""
    dims = _check_dims(dims)
    vf = pattern.target_volume_fraction
    if pattern.kind in ("p", "d", "g", "iwp"):
        rho = _by_rank(_level_set(pattern.kind, dims), vf)
    elif pattern.kind == "ball":
        cs = [(np.arange(n) + 0.5) / n - 0.5 for n in dims]
        X, Y, Z = np.meshgrid(*cs, indexing="ij")
        rho = _by_rank(np.sqrt(X ** 2 + Y ** 2 + Z ** 2), vf)
    else:
        base = np.random.default_rng(pattern.seed).uniform(0.3, 0.7, size=dims)
        lo, hi = -1.0, 1.0
        for _ in range(60):
            mid = 0.5 * (lo + hi)
            if np.clip(base + mid, PATTERN_FLOOR, 1.0).mean(dtype=np.float64) < vf:
                lo = mid
            else:
                hi = mid
        rho = np.clip(base + 0.5 * (lo + hi), PATTERN_FLOOR, 1.0)
    mean = rho.mean(dtype=np.float64)
    if abs(mean - vf) > 0.01:
        raise ValueError(f"volume fraction {vf} unattainable for pattern {pattern.kind!r} "
                         f"on grid {dims} (reached {mean:.4f})")
    return DensityField(dims, rho, np.zeros(dims))


def _filter(fld_dims, spec: FilterSpec, arr, adjoint: int):
    if spec.kernel is not None:
        raise NotImplementedError("custom filter kernels are not supported on the device path; "
                                  "use the cone kernel (FilterSpec(radius))")
    src, host = _dev.to_device(arr, shape=fld_dims)
    ctx = _dev.shared_context(fld_dims, radius=spec.radius)
    out = ctx.empty(*fld_dims)
    ctx.call("otm_filter", _dev.ptr(src), _dev.ptr(out), adjoint)
    return _dev.like_input(out, host)


def filter_forward(fld: DensityField, spec: FilterSpec):
    """rho_f = F rho, periodic cone filter (field.py:230-233), on the device."""
    return _filter(tuple(fld.dims), spec, fld.rho, 0)


def filter_backward(fld: DensityField, spec: FilterSpec, grad_wrt_filtered):
    """Exact adjoint F^T g (field.py:236-243), on the device."""
    shape = tuple(grad_wrt_filtered.shape)
    if shape != tuple(fld.dims):
        raise ValueError(f"gradient shape {shape} != field shape {tuple(fld.dims)}")
    return _filter(tuple(fld.dims), spec, grad_wrt_filtered, 1)


def project_central_symmetry(fld: DensityField, also_grad: bool = False) -> None:
    """Average with the point-symmetric partner, in place (field.py:246-255)."""
    for name in (("rho", "grad") if also_grad else ("rho",)):
        arr = getattr(fld, name)
        t, host = _dev.to_device(arr, shape=tuple(fld.dims))
        ctx = _dev.shared_context(tuple(fld.dims))
        ctx.call("otm_symmetrize", _dev.ptr(t))
        if host:
            arr[...] = t.cpu().numpy()
        else:
            arr.copy_(t)
