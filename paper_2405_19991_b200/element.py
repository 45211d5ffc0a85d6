"""Unit-voxel element constants and SIMP interpolation (reference: element.py).

These are host-side constants of the API; the device kernels hard-code the same
template (K0 = (5 I + N1 - J) / 12, f0 = +-1/4) and evaluate SIMP inside the
fused filter sweep.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

#: corner n at (n & 1, (n >> 1) & 1, (n >> 2) & 1)  (element.py:16-18)
CORNERS = np.array([[(n >> a) & 1 for a in range(3)] for n in range(8)], dtype=np.int64)


@dataclass(frozen=True)
class ElementTemplates:
    """K0 (8x8), T0 (8x3 corner coordinates), f0 = K0 @ T0  (element.py:21-39)."""
    K0: np.ndarray
    T0: np.ndarray
    f0: np.ndarray


@dataclass(frozen=True)
class MaterialParams:
    """Two-phase SIMP material (element.py:42-56)."""
    kappa0: float = 1.0
    kappa_min: float = 1e-4
    penalty: float = 3.0

    def __post_init__(self):
        if not (self.kappa0 > self.kappa_min > 0.0):
            raise ValueError(f"need kappa0 > kappa_min > 0, got {self.kappa0}, {self.kappa_min}")
        if self.penalty < 1.0:
            raise ValueError(f"penalty must be >= 1, got {self.penalty}")


def template_matrix(axis_scale=(1.0, 1.0, 1.0)) -> np.ndarray:
    """K[a, b] = sum_ax s_ax * stiff(ax) * mass * mass; depends on a ^ b only."""
    st, ms = (1.0, -1.0), (1.0 / 3.0, 1.0 / 6.0)
    kt = np.zeros(8)
    for d in range(8):
        for ax in range(3):
            term = axis_scale[ax]
            for q in range(3):
                bit = (d >> q) & 1
                term *= st[bit] if q == ax else ms[bit]
            kt[d] += term
    idx = np.arange(8)
    return kt[idx[:, None] ^ idx[None, :]]


def build_templates() -> ElementTemplates:
    """element.py:72-88 (closed form instead of Gauss quadrature; identical values)."""
    K0 = template_matrix()
    T0 = CORNERS.astype(np.float64)
    return ElementTemplates(K0=K0, T0=T0, f0=K0 @ T0)


def simp_conductivity(rho_filtered, params: MaterialParams):
    """kappa_min + rho^p (kappa0 - kappa_min)  (element.py:91-94)."""
    r = rho_filtered
    if not hasattr(r, "data_ptr"):
        r = np.asarray(r, dtype=np.float64)
    return params.kappa_min + r ** params.penalty * (params.kappa0 - params.kappa_min)


def simp_derivative(rho_filtered, params: MaterialParams):
    """p rho^(p-1) (kappa0 - kappa_min)  (element.py:97-100)."""
    r = rho_filtered
    if not hasattr(r, "data_ptr"):
        r = np.asarray(r, dtype=np.float64)
    return params.penalty * r ** (params.penalty - 1.0) * (params.kappa0 - params.kappa_min)
