"""Homogenized conductivity and its density gradient (reference: homogenize.py).

The three unit-gradient cases are solved batched on the device; the tensor and
the sensitivities are fixed-order fp64 reductions over per-element energies that
are recomputed from the corrective fields (nothing per element is cached).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _dev
from .element import MaterialParams
from .solver import GridHierarchy

PACKED_PAIRS = ((0, 0), (1, 1), (2, 2), (0, 1), (1, 2), (0, 2))     # homogenize.py:23
PACKED_NAMES = ("k11", "k22", "k33", "k12", "k23", "k13")


@dataclass(frozen=True)
class ConductivityTensor:
    """Symmetric 3x3 packed as [k11, k22, k33, k12, k23, k13] (homogenize.py:27-55)."""

    vec: np.ndarray

    def __post_init__(self):
        v = np.asarray(self.vec, dtype=np.float64).reshape(-1)
        if v.size != 6:
            raise ValueError(f"expected 6 packed components, got {v.size}")
        object.__setattr__(self, "vec", v)

    @classmethod
    def from_matrix(cls, m) -> "ConductivityTensor":
        m = np.asarray(m, dtype=np.float64)
        if m.shape != (3, 3) or not np.allclose(m, m.T, atol=1e-12):
            raise ValueError("expected a symmetric 3x3 matrix")
        return cls(np.array([m[0, 0], m[1, 1], m[2, 2], m[0, 1], m[1, 2], m[0, 2]]))

    def as_matrix(self) -> np.ndarray:
        k11, k22, k33, k12, k23, k13 = self.vec
        return np.array([[k11, k12, k13], [k12, k22, k23], [k13, k23, k33]])

    def is_positive_definite(self) -> bool:
        try:
            np.linalg.cholesky(self.as_matrix())
            return True
        except np.linalg.LinAlgError:
            return False


@dataclass
class HomogenizationResult:
    """Tensor + corrective fields (homogenize.py:58-68).  ``pair_energy`` and
    ``elem_diff`` are materialised on first access (the device path never stores
    them)."""

    tensor: ConductivityTensor
    T_fields: list
    rho_filtered: object
    params: MaterialParams
    vcycles: int = 0
    _hier: Optional[GridHierarchy] = field(default=None, repr=False)
    _version: int = field(default=-1, repr=False)
    _cache: dict = field(default_factory=dict, repr=False)

    def _host(self):
        return not hasattr(self.rho_filtered, "data_ptr")

    def _activate(self):
        """Make the hierarchy hold this result's factors and fields again."""
        h = self._hier
        if h.ctx.version != self._version:
            h.build_density(self.rho_filtered, self.params)
            T3 = _stack_fields(self.T_fields, h.dims)
            h.ctx.call("otm_set_warm", _dev.ptr(T3))
            h.ctx.version += 1
            self._version = h.ctx.version

    @property
    def pair_energy(self):
        if "E" not in self._cache:
            self._activate()
            h = self._hier
            E = _dev.torch().empty((6,) + h.dims, dtype=_dev.torch().float64, device="cuda")
            h.ctx.call("otm_pair_energy", _dev.ptr(E))
            self._cache["E"] = E.cpu().numpy() if self._host() else E
        return self._cache["E"]

    @property
    def elem_diff(self):
        """Per case (nx, ny, nz, 8) float32: c_a[i] - T_i[e + c_a] (homogenize.py:94-100)."""
        if "w" not in self._cache:
            t = _dev.torch()
            h = self._hier
            out = []
            for i, T in enumerate(self.T_fields):
                Td, _ = _dev.to_device(T, shape=h.dims)
                Td = Td.contiguous()
                w = t.empty(tuple(h.dims) + (8,), dtype=t.float32, device="cuda")
                h.ctx.call("otm_elem_diff", _dev.ptr(Td), i, _dev.ptr(w))
                out.append(w.cpu().numpy() if self._host() else w)
            self._cache["w"] = out
        return self._cache["w"]


def _stack_fields(fields, dims):
    t = _dev.torch()
    parts = [_dev.to_device(f, shape=dims)[0] for f in fields]
    return t.stack(parts).contiguous()


def solve_cases(hier: GridHierarchy, rho_filtered, params: MaterialParams, tol: float = 1e-6,
                max_vcycles: int = 200, warm: Optional[Sequence] = None):
    """SIMP + build + the three load cases (homogenize.py:71-91), batched."""
    host = not hasattr(rho_filtered, "data_ptr")
    hier.build_density(rho_filtered, params)
    W = _stack_fields(warm, hier.dims) if warm is not None else None
    T, cycles, _ = hier.solve3(None, tol=tol, max_vcycles=max_vcycles, warm=W)
    fields = [T[i].cpu().numpy() for i in range(3)] if host else [T[i] for i in range(3)]
    return fields, cycles


def effective_tensor(hier: GridHierarchy, T_fields: Sequence, rho_filtered, params: MaterialParams,
                     vcycles: int = 0) -> HomogenizationResult:
    """kappa^H_c = sum_e kappa_e E_c[e] / M (homogenize.py:103-130)."""
    hier.build_density(rho_filtered, params)
    T3 = _stack_fields(T_fields, hier.dims)
    hier.ctx.call("otm_set_warm", _dev.ptr(T3))
    out = (C.c_double * 6)()
    hier.ctx.call("otm_tensor", out)
    hier.ctx.version += 1
    return HomogenizationResult(tensor=ConductivityTensor(np.array(out[:])), T_fields=list(T_fields),
                                rho_filtered=rho_filtered, params=params, vcycles=vcycles, _hier=hier,
                                _version=hier.ctx.version)


def homogenize(hier: GridHierarchy, rho_filtered, params: MaterialParams, tol: float = 1e-6,
               max_vcycles: int = 200, warm: Optional[Sequence] = None) -> HomogenizationResult:
    """solve_cases + effective_tensor (homogenize.py:133-140) without a host round trip."""
    host = not hasattr(rho_filtered, "data_ptr")
    hier.build_density(rho_filtered, params)
    W = _stack_fields(warm, hier.dims) if warm is not None else None
    T, cycles, _ = hier.solve3(None, tol=tol, max_vcycles=max_vcycles, warm=W)
    out = (C.c_double * 6)()
    hier.ctx.call("otm_tensor", out)
    fields = [T[i].cpu().numpy() for i in range(3)] if host else [T[i] for i in range(3)]
    return HomogenizationResult(tensor=ConductivityTensor(np.array(out[:])), T_fields=fields,
                                rho_filtered=rho_filtered, params=params, vcycles=cycles, _hier=hier,
                                _version=hier.ctx.version)


def tensor_sensitivity(result: HomogenizationResult, dG_dkappa):
    """d g / d rho_f = kappa'(rho_f) (dG . E) / M  (homogenize.py:143-160)."""
    dG = np.asarray(dG_dkappa, dtype=np.float64).reshape(-1)
    if dG.size != 6:
        raise ValueError(f"expected 6 objective weights, got {dG.size}")
    if result._hier is None:
        raise RuntimeError("homogenization caches missing; run effective_tensor first")
    result._activate()
    h = result._hier
    sens = h.ctx.empty(*h.dims)
    h.ctx.call("otm_sensitivity", (C.c_double * 6)(*dG), _dev.ptr(sens))
    return sens.cpu().numpy() if result._host() else sens
