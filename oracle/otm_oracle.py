"""CPU oracle for the OpenTM homogenization + OC hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2405_19991_b200`` imports this
module: it is the checker that ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` run against the
CUDA product path.  It is never the thing measured as the product and never a
fallback.

It is an independent numpy restatement of the reference package
(``/root/reference/pkg/src/opentm``, abbreviated ``src/`` below).  Each
function cites the reference ``file:line`` whose behaviour it restates.  The
algorithm is the reference's own: fp64 fields, an 8-colour Gauss-Seidel
V-cycle iterated until the fp64 relative residual reaches ``tol``, the cone
density filter, the adaptive-volume OC loop.  Summation orders differ from the
reference, so agreement is to round-off, not bit-for-bit.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference in the
build container (where ``/root/reference`` exists) and stores its outputs in
``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this module
against every one of those vectors.  (SciPy is the reference's only numeric
dependency besides numpy - ``pkg/pyproject.toml:5-10`` - and this module uses
the same ``scipy.sparse.linalg.splu`` for the largest coarse levels.)
"""

from __future__ import annotations

import math
import time
import warnings
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

# --------------------------------------------------------------------------
# element: src/element.py
# --------------------------------------------------------------------------

#: corner n of the unit voxel sits at (n&1, (n>>1)&1, (n>>2)&1)  (src/element.py:16-18)
CORNER_BITS = np.array([[(n >> ax) & 1 for ax in range(3)] for n in range(8)], dtype=np.int64)

_STIFF_1D = ((1.0, -1.0), (-1.0, 1.0))
_MASS_1D = ((1.0 / 3.0, 1.0 / 6.0), (1.0 / 6.0, 1.0 / 3.0))


def voxel_template(axis_scale=(1.0, 1.0, 1.0)) -> np.ndarray:
    """8x8 trilinear conduction matrix, sum over axes of stiffness x mass x mass.

    Restates ``_axis_template``/``_level_template`` (src/solver.py:43-54); with unit
    scales it is the element matrix K0 of ``build_templates`` (src/element.py:72-88)."""
    K = np.zeros((8, 8))
    for a in range(8):
        for b in range(8):
            acc = 0.0
            for ax in range(3):
                term = axis_scale[ax]
                for q in range(3):
                    tab = _STIFF_1D if q == ax else _MASS_1D
                    term *= tab[CORNER_BITS[a, q]][CORNER_BITS[b, q]]
                acc += term
            K[a, b] = acc
    return K


K0 = voxel_template()
#: unit-gradient loads f0 = K0 @ corner coordinates (src/element.py:86)
F0 = K0 @ CORNER_BITS.astype(np.float64)


@dataclass(frozen=True)
class Material:
    """SIMP parameters (src/element.py:42-56)."""
    kappa0: float = 1.0
    kappa_min: float = 1e-4
    penalty: float = 3.0


def simp(rho, mat: Material):
    """kappa = kmin + rho^p (k0 - kmin)  (src/element.py:91-94)."""
    r = np.asarray(rho, dtype=np.float64)
    return mat.kappa_min + r ** mat.penalty * (mat.kappa0 - mat.kappa_min)


def simp_prime(rho, mat: Material):
    """d kappa / d rho = p rho^(p-1) (k0 - kmin)  (src/element.py:97-100)."""
    r = np.asarray(rho, dtype=np.float64)
    return mat.penalty * r ** (mat.penalty - 1.0) * (mat.kappa0 - mat.kappa_min)


# --------------------------------------------------------------------------
# field: src/field.py
# --------------------------------------------------------------------------

def filter_taps(radius: float = 1.5):
    """Cone taps max(0, r - |o|) on the cube of reach ceil(r)-1, normalised.

    src/field.py:60-93.  Returned in lexicographic (dx, dy, dz) order."""
    reach = int(math.ceil(radius)) - 1
    offs, wts = [], []
    for dx in range(-reach, reach + 1):
        for dy in range(-reach, reach + 1):
            for dz in range(-reach, reach + 1):
                w = max(0.0, radius - math.sqrt(dx * dx + dy * dy + dz * dz))
                if w > 0.0:
                    offs.append((dx, dy, dz))
                    wts.append(w)
    wts = np.array(wts)
    return np.array(offs, dtype=np.int64), wts / wts.sum()


def _shifted(a: np.ndarray, off) -> np.ndarray:
    """b[v] = a[v + off] with periodic wrap."""
    return np.roll(a, tuple(-int(o) for o in off), axis=(0, 1, 2))


def filter_fwd(rho: np.ndarray, radius: float = 1.5) -> np.ndarray:
    """rho_f[v] = sum_k w_k rho[v + o_k]  (src/field.py:222-233)."""
    offs, w = filter_taps(radius)
    out = np.zeros_like(rho, dtype=np.float64)
    for o, wk in zip(offs, w):
        out += wk * _shifted(rho, o)
    return out


def filter_adj(g: np.ndarray, radius: float = 1.5) -> np.ndarray:
    """Exact adjoint: sum_k w_k g[v - o_k]  (src/field.py:236-243)."""
    offs, w = filter_taps(radius)
    out = np.zeros_like(g, dtype=np.float64)
    for o, wk in zip(offs, w):
        out += wk * _shifted(g, -o)
    return out


def central_symmetrize(a: np.ndarray) -> np.ndarray:
    """0.5 (a + a[::-1,::-1,::-1])  (src/field.py:246-255)."""
    return 0.5 * (a + a[::-1, ::-1, ::-1])


PATTERN_FLOOR = 0.001  # src/field.py:18


def _cell_angles(dims):
    grids = [2.0 * np.pi * (np.arange(n) + 0.5) / n for n in dims]
    return np.meshgrid(*grids, indexing="ij")


def _tpms(kind: str, dims) -> np.ndarray:
    """Level-set generators (src/field.py:141-160)."""
    X, Y, Z = _cell_angles(dims)
    cx, cy, cz = np.cos(X), np.cos(Y), np.cos(Z)
    sx, sy, sz = np.sin(X), np.sin(Y), np.sin(Z)
    if kind == "p":
        return cx + cy + cz
    if kind == "g":
        return sx * cy + sy * cz + sz * cx
    if kind == "d":
        return sx * sy * sz + sx * cy * cz + cx * sy * cz + cx * cy * sz
    if kind == "iwp":
        return 2.0 * (cx * cy + cy * cz + cz * cx) - (np.cos(2 * X) + np.cos(2 * Y) + np.cos(2 * Z))
    raise ValueError(kind)


def _rank_select(values: np.ndarray, vf: float) -> np.ndarray:
    """Largest-generator voxels become solid, the rest PATTERN_FLOOR (src/field.py:163-176)."""
    n = values.size
    count = int(round(n * (vf - PATTERN_FLOOR) / (1.0 - PATTERN_FLOOR)))
    count = min(max(count, 0), n)
    order = np.argsort(values.ravel(), kind="stable")[::-1]
    flat = np.full(n, PATTERN_FLOOR)
    flat[order[:count]] = 1.0
    return flat.reshape(values.shape)


def seed_density(dims, kind: str = "iwp", vf: float = 0.5, seed: int = 0) -> np.ndarray:
    """Seed patterns of ``init_density`` (src/field.py:192-219)."""
    dims = tuple(int(n) for n in dims)
    kind = {"centerball": "ball"}.get(kind.lower(), kind.lower())
    if kind in ("p", "d", "g", "iwp"):
        rho = _rank_select(_tpms(kind, dims), vf)
    elif kind == "ball":
        c = [(np.arange(n) + 0.5) / n - 0.5 for n in dims]
        X, Y, Z = np.meshgrid(*c, indexing="ij")
        rho = _rank_select(np.sqrt(X * X + Y * Y + Z * Z), vf)
    elif kind == "random":
        base = np.random.default_rng(seed).uniform(0.3, 0.7, size=dims)
        lo, hi = -1.0, 1.0
        for _ in range(60):
            mid = 0.5 * (lo + hi)
            if np.clip(base + mid, PATTERN_FLOOR, 1.0).mean(dtype=np.float64) < vf:
                lo = mid
            else:
                hi = mid
        rho = np.clip(base + 0.5 * (lo + hi), PATTERN_FLOOR, 1.0)
    else:
        raise ValueError(f"unknown pattern {kind!r}")
    if abs(rho.mean() - vf) > 0.01:
        raise ValueError("volume fraction unattainable")
    return rho


# --------------------------------------------------------------------------
# solver: src/solver.py
# --------------------------------------------------------------------------

class ConvergenceFailure(RuntimeError):
    """Mirror of ConvergenceError (src/solver.py:35-40)."""

    def __init__(self, msg, residual):
        super().__init__(msg)
        self.residual = residual


def level_chain(dims, coarse_target=64, direct_limit=40000):
    """Halve every axis > 1 while the product exceeds ``coarse_target`` and all such
    axes are even (src/solver.py:217-231).  Returns [(dims, axis_scale), ...]."""
    dims = tuple(int(n) for n in dims)
    if len(dims) != 3 or min(dims) < 1:
        raise ValueError(f"bad dims {dims}")
    chain = [dims]
    while int(np.prod(chain[-1])) > coarse_target and all(n % 2 == 0 for n in chain[-1] if n > 1):
        chain.append(tuple(n // 2 if n > 1 else 1 for n in chain[-1]))
    if int(np.prod(chain[-1])) > direct_limit:
        raise ValueError(f"dims {dims} do not coarsen below {direct_limit} vertices")
    # per-axis scale norm*vol/h^2 (src/solver.py:233-245)
    out = []
    h = [1.0, 1.0, 1.0]
    norm = 1.0
    for li, d in enumerate(chain):
        vol = h[0] * h[1] * h[2]
        out.append((d, tuple(norm * vol / (h[a] * h[a]) for a in range(3))))
        if li + 1 < len(chain):
            nxt = chain[li + 1]
            for a in range(3):
                if nxt[a] < d[a]:
                    h[a] *= 2.0
                    norm *= 0.5
    return out


def _offsets27():
    return [(dx, dy, dz) for dx in (-1, 0, 1) for dy in (-1, 0, 1) for dz in (-1, 0, 1)]


def _canon(d, dims):
    # an offset of -1 on a length-2 axis is the same neighbour as +1, and any
    # offset on a length-1 axis is the vertex itself (src/solver.py:57-63)
    out = []
    for s, n in zip(d, dims):
        if n == 1:
            out.append(0)
        elif n == 2 and s == -1:
            out.append(1)
        else:
            out.append(s)
    return tuple(out)


class Level:
    """Per-level element factors and 27-point stencil coefficients (src/solver.py:66-108)."""

    def __init__(self, dims, axis_scale):
        self.dims = tuple(dims)
        self.axis_scale = tuple(axis_scale)
        self.template = voxel_template(axis_scale)
        self.kappa = None
        self.coef = None  # {offset: array}
        self.T = np.zeros(self.dims)
        self.f = np.zeros(self.dims)
        self.r = np.zeros(self.dims)

    def set_kappa(self, kappa):
        kappa = np.asarray(kappa, dtype=np.float64)
        if kappa.shape != self.dims:
            raise ValueError("kappa shape mismatch")
        self.kappa = kappa
        # vertex v is corner a of element v - c_a; it couples to corner b, v + (c_b - c_a)
        elem_at = [np.roll(kappa, tuple(CORNER_BITS[a]), axis=(0, 1, 2)) for a in range(8)]
        coef = {}
        for a in range(8):
            for b in range(8):
                d = _canon(tuple(int(x) for x in CORNER_BITS[b] - CORNER_BITS[a]), self.dims)
                term = self.template[a, b] * elem_at[a]
                coef[d] = coef[d] + term if d in coef else term
        self.coef = coef
        if not (coef[(0, 0, 0)] > 0).all():
            raise RuntimeError("non-positive diagonal")

    def apply(self, T):
        """(K T)[v] = sum_d W_d[v] T[v+d]  (src/solver.py:111-119)."""
        out = self.coef[(0, 0, 0)] * T
        for d, W in self.coef.items():
            if d != (0, 0, 0):
                out = out + W * _shifted(T, d)
        return out


class Hierarchy:
    """Multigrid level stack + coarsest direct solve (src/solver.py:203-338)."""

    def __init__(self, dims, coarse_target=64, direct_limit=40000, sweeps=(1, 1)):
        self.levels = [Level(d, s) for d, s in level_chain(dims, coarse_target, direct_limit)]
        self.pre, self.post = sweeps
        self._coarse = None
        self.history = []

    @property
    def dims(self):
        return self.levels[0].dims

    def build(self, kappa):
        """Child-mean kappa per level, then factor the coarsest (src/solver.py:257-305)."""
        kap = np.asarray(kappa, dtype=np.float64)
        for li, lev in enumerate(self.levels):
            if li > 0:
                fine = self.levels[li - 1].dims
                for ax in range(3):
                    if lev.dims[ax] < fine[ax]:
                        shp = list(kap.shape)
                        shp[ax:ax + 1] = [shp[ax] // 2, 2]
                        kap = kap.reshape(shp).mean(axis=ax + 1)
            lev.set_kappa(kap)
        self._factor()

    def _factor(self):
        lev = self.levels[-1]
        n = int(np.prod(lev.dims))
        if n == 1:
            self._coarse = None
            return
        idx = np.arange(n).reshape(lev.dims)
        rows, cols, vals = [], [], []
        for d, W in lev.coef.items():
            rows.append(idx.ravel())
            cols.append(_shifted(idx, d).ravel())
            vals.append(W.ravel())
        from scipy.sparse import coo_matrix
        A = coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                       shape=(n, n)).tocsc()
        red = A[1:, 1:]
        if n <= 4096:
            self._coarse = ("dense", np.linalg.inv(red.toarray()))
        else:
            from scipy.sparse.linalg import splu
            self._coarse = ("lu", splu(red.tocsc()))

    def coarse(self):
        """Pinned direct solve with the mean projected out (src/solver.py:307-324)."""
        lev = self.levels[-1]
        f = lev.f.ravel().astype(np.float64)
        tot, mag = f.sum(), np.abs(f).sum()
        if mag > 0 and abs(tot) > 1e-4 * mag:
            warnings.warn("coarse load has a nonzero mean component", RuntimeWarning)
        f = f - tot / f.size
        x = np.zeros_like(f)
        if self._coarse is not None:
            kind, fac = self._coarse
            x[1:] = fac @ f[1:] if kind == "dense" else fac.solve(f[1:])
        x -= x.mean()
        lev.T[...] = x.reshape(lev.dims)

    def vcycle(self):
        """src/solver.py:326-338."""
        L = len(self.levels) - 1
        for li in range(L):
            lev = self.levels[li]
            if li:
                lev.T[...] = 0.0
            gauss_seidel8(lev, self.pre)
            lev.r[...] = lev.f - lev.apply(lev.T)
            restrict_fw(lev, self.levels[li + 1])
        self.coarse()
        for li in range(L - 1, -1, -1):
            prolong_add(self.levels[li], self.levels[li + 1])
            gauss_seidel8(self.levels[li], self.post)


def gauss_seidel8(lev: Level, sweeps=1):
    """Parity-coloured Gauss-Seidel, colours in lexicographic order (src/solver.py:122-164)."""
    dims = lev.dims
    if any(n > 1 and n % 2 for n in dims):
        raise ValueError(f"relaxation needs even axes, got {dims}")
    ncol = [min(2, n) for n in dims]
    colours = [(a, b, c) for a in range(ncol[0]) for b in range(ncol[1]) for c in range(ncol[2])]
    diag = lev.coef[(0, 0, 0)]
    for _ in range(sweeps):
        for col in colours:
            sel = tuple(slice(c, None, 2) for c in col)
            acc = lev.f[sel].copy()
            for d, W in lev.coef.items():
                if d == (0, 0, 0):
                    continue
                src, shift = [], []
                for ax in range(3):
                    t = col[ax] + d[ax]
                    par = t % 2 if dims[ax] > 1 else 0
                    src.append(slice(par, None, 2))
                    shift.append(-((t - par) // 2))
                nb = lev.T[tuple(src)]
                if any(shift):
                    nb = np.roll(nb, tuple(shift), axis=(0, 1, 2))
                acc -= W[sel] * nb
            lev.T[sel] = acc / diag[sel]


def restrict_fw(fine: Level, coarse: Level):
    """[1/4, 1/2, 1/4] per coarsened axis then even subsample (src/solver.py:167-177)."""
    s = fine.r
    pick = []
    for ax in range(3):
        if coarse.dims[ax] < fine.dims[ax]:
            s = 0.5 * s + 0.25 * (np.roll(s, 1, axis=ax) + np.roll(s, -1, axis=ax))
            pick.append(slice(0, None, 2))
        else:
            pick.append(slice(None))
    coarse.f[...] = s[tuple(pick)]


def prolong_add(fine: Level, coarse: Level):
    """Trilinear interpolation of the coarse T added to the fine T (src/solver.py:180-200)."""
    t = coarse.T
    for ax in range(3):
        if coarse.dims[ax] < fine.dims[ax]:
            shp = list(t.shape)
            shp[ax] *= 2
            u = np.empty(shp)
            ev = [slice(None)] * 3
            od = [slice(None)] * 3
            ev[ax] = slice(0, None, 2)
            od[ax] = slice(1, None, 2)
            u[tuple(ev)] = t
            u[tuple(od)] = 0.5 * (t + np.roll(t, -1, axis=ax))
            t = u
    fine.T += t


def macro_load(hier: Hierarchy, case: int) -> np.ndarray:
    """f_i[v] = sum_a f0[a,i] kappa[v - c_a]  (src/solver.py:347-363)."""
    lev = hier.levels[0]
    f0 = lev.template @ CORNER_BITS.astype(np.float64)
    out = np.zeros(lev.dims)
    for a in range(8):
        out += f0[a, case] * np.roll(lev.kappa, tuple(CORNER_BITS[a]), axis=(0, 1, 2))
    return out


def solve(hier: Hierarchy, f: np.ndarray, tol=1e-6, max_cycles=200, x0=None):
    """V-cycle iteration to ||f - K T|| / ||f|| <= tol  (src/solver.py:366-406)."""
    lev = hier.levels[0]
    if f.shape != lev.dims:
        raise ValueError("load shape mismatch")
    fnorm = float(np.linalg.norm(f))
    hier.history = []
    if fnorm == 0.0:
        lev.T[...] = 0.0
        return lev.T.copy(), 0
    lev.f[...] = f - f.mean()
    lev.T[...] = 0.0 if x0 is None else (x0 - x0.mean())
    rel = np.inf
    for cyc in range(1, max_cycles + 1):
        hier.vcycle()
        lev.T -= lev.T.mean()
        rel = float(np.linalg.norm(lev.f - lev.apply(lev.T))) / fnorm
        hier.history.append(rel)
        if rel <= tol:
            return lev.T.copy(), cyc
    raise ConvergenceFailure(f"no convergence after {max_cycles} V-cycles ({rel:.3e})", rel)


# --------------------------------------------------------------------------
# homogenize / objective: src/homogenize.py, src/objective.py
# --------------------------------------------------------------------------

PAIRS = ((0, 0), (1, 1), (2, 2), (0, 1), (1, 2), (0, 2))  # src/homogenize.py:23


def solve_three(hier: Hierarchy, rho_f, mat: Material, tol=1e-6, max_cycles=200, warm=None):
    """src/homogenize.py:71-91."""
    hier.build(simp(rho_f, mat))
    Ts, total = [], 0
    for i in range(3):
        T, c = solve(hier, macro_load(hier, i), tol, max_cycles, None if warm is None else warm[i])
        Ts.append(T)
        total += c
    return Ts, total


def pair_energies(T_fields) -> np.ndarray:
    """E_c[e] = w_i . K0 w_j with w_i[e,a] = c_a[i] - T_i[e + c_a]  (src/homogenize.py:94-130)."""
    W = []
    for i, T in enumerate(T_fields):
        w = np.stack([CORNER_BITS[a, i] - _shifted(np.asarray(T, np.float64), CORNER_BITS[a])
                      for a in range(8)], axis=-1)
        W.append(w)
    KW = [w @ K0 for w in W]
    return np.stack([np.einsum("...a,...a->...", W[i], KW[j]) for i, j in PAIRS])


def tensor_from_energies(E, rho_f, mat: Material) -> np.ndarray:
    kap = simp(rho_f, mat)
    return np.array([float((kap * E[c]).sum()) / kap.size for c in range(6)])


def sensitivity(E, rho_f, dG, mat: Material) -> np.ndarray:
    """dG . E * kappa'(rho_f) / M  (src/homogenize.py:143-160)."""
    dG = np.asarray(dG, dtype=np.float64).reshape(6)
    return simp_prime(rho_f, mat) * np.tensordot(dG, E, axes=1) / rho_f.size


def objective(kind: str, target, k):
    """mse / rel / l1 with NaN targets masked (src/objective.py:48-72)."""
    t = np.asarray(target, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    m = ~np.isnan(t)
    if kind == "mse":
        d = np.where(m, k - t, 0.0)
        return float((d * d).sum()), 2.0 * d
    if kind == "rel":
        tt = np.where(m, t, 1.0)
        d = np.where(m, k / tt - 1.0, 0.0)
        return float((d * d).sum()), np.where(m, 2.0 * d / tt, 0.0)
    d = np.where(m, k - t, 0.0)
    return float(np.abs(d).sum()), np.sign(d)


# --------------------------------------------------------------------------
# optimize: src/optimize.py
# --------------------------------------------------------------------------

@dataclass
class Governor:
    """Adaptive volume ceiling (src/optimize.py:38-54)."""
    vstar: float = 1.0
    df: float = 1.0
    gap: float = 0.0
    count: int = 0
    bound: float = 1e-4
    iter: int = 0
    g_prev: float = 1.0
    reduced: bool = False

    @property
    def pending_decrease(self):
        return self.gap * self.df if self.reduced else math.inf


def governor_step(st: Governor, g: float, mean_rho: float, mean_rho_p: float) -> float:
    """Algorithm 1 of the paper as coded in src/optimize.py:57-86."""
    if g <= st.bound:
        st.gap = st.vstar - mean_rho_p
        st.vstar -= st.gap * st.df
        st.df *= 0.8
        st.reduced = True
    stalled = abs(st.g_prev - g) < max(0.1 * g, 1e-7)
    if stalled and g > st.bound and mean_rho > st.vstar - 0.01:
        st.count += 1
    else:
        st.count = 0
    if st.count >= 5:
        st.vstar += 0.3 * st.gap * st.df
        st.count = 0
    st.g_prev = g
    st.iter += 1
    return st.vstar


@dataclass(frozen=True)
class OC:
    """src/optimize.py:89-111."""
    min_density: float = 0.001
    step_limit: float = 0.02
    damp: float = 0.5
    bisection_tol: float = 1e-5


def oc_step(rho, sens, vol_bound, p: OC = OC()):
    """Move-limited multiplicative update with lambda bisection (src/optimize.py:114-160)."""
    rho = np.asarray(rho, dtype=np.float64)
    sens = np.asarray(sens, dtype=np.float64)
    if rho.shape != sens.shape:
        raise ValueError("shape mismatch")
    lo = np.maximum(rho - p.step_limit, p.min_density)
    hi = np.minimum(rho + p.step_limit, 1.0)
    desc = rho.size * (-sens)

    def trial(lam):
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            return np.clip(rho * np.maximum(desc / lam, 1e-10) ** p.damp, lo, hi)

    slack = np.where(desc > 0.0, hi, np.where(desc < 0.0, lo, rho))
    if float(slack.mean()) <= vol_bound:
        return slack, {"lam": 0.0, "active": False, "evals": 1}
    evals = 1
    a, b = 1e-30, 1.0
    for _ in range(200):
        evals += 1
        if float(trial(b).mean()) <= vol_bound:
            break
        b *= 4.0
    while (b - a) / (a + b) > 1e-13:
        mid = 0.5 * (a + b)
        cur = trial(mid)
        evals += 1
        m = float(cur.mean())
        if m > vol_bound:
            a = mid
        else:
            b = mid
        if abs(m - vol_bound) <= p.bisection_tol:
            break
    lam = 0.5 * (a + b)
    return trial(lam), {"lam": lam, "active": True, "evals": evals + 1}


@dataclass
class Record:
    """IterationRecord (src/optimize.py:222-230)."""
    iter: int
    g: float
    volfrac: float
    volfrac_filtered: float
    vstar: float
    vcycles: int
    ms: float


@dataclass
class Run:
    """The subset of RunConfig (src/optimize.py:171-219) on the hot path (model 'oc')."""
    dims: tuple
    target: Sequence[float]
    objective: str = "mse"
    material: Material = field(default_factory=Material)
    radius: float = 1.5
    init: tuple = ("iwp", 0.5, 0)
    init_field: Optional[np.ndarray] = None
    oc: OC = field(default_factory=OC)
    max_iter: int = 500
    conv_threshold: float = 1e-4
    symmetry: str = "none"
    solver_tol: float = 1e-6
    max_vcycles: int = 200
    governor_bound: float = 1e-4


def optimize(cfg: Run, callback: Optional[Callable] = None):
    """Adaptive-volume OC loop (src/optimize.py:257-379), model 'oc' only.

    Returns (rho, kappa_h, log, converged)."""
    rho = (np.array(cfg.init_field, dtype=np.float64) if cfg.init_field is not None
           else seed_density(cfg.dims, *cfg.init))
    if cfg.symmetry == "central":
        rho = central_symmetrize(rho)
    hier = Hierarchy(cfg.dims)
    gov = Governor(bound=cfg.governor_bound)
    log, warm, plateau, g_last, converged, kh = [], None, 0, None, False, None
    for it in range(1, cfg.max_iter + 1):
        t0 = time.perf_counter()
        rho_f = filter_fwd(rho, cfg.radius)
        Ts, cycles = solve_three(hier, rho_f, cfg.material, cfg.solver_tol, cfg.max_vcycles, warm)
        warm = Ts
        E = pair_energies(Ts)
        kh = tensor_from_energies(E, rho_f, cfg.material)
        g, dG = objective(cfg.objective, cfg.target, kh)
        sens = filter_adj(sensitivity(E, rho_f, dG, cfg.material), cfg.radius)
        if cfg.symmetry == "central":
            sens = central_symmetrize(sens)
        log.append(Record(it, g, float(rho.mean()), float(rho_f.mean()), gov.vstar, cycles,
                          (time.perf_counter() - t0) * 1e3))
        if callback is not None:
            callback(it, rho, kh, g)
        plateau = plateau + 1 if (g_last is not None and abs(g - g_last) < cfg.conv_threshold) else 0
        g_last = g
        if g <= 1e-12:
            converged = True
        elif plateau >= 3:
            converged = gov.pending_decrease < 1e-4 and g <= gov.bound
        if converged or it == cfg.max_iter:
            break
        mean_now = float(rho.mean())
        vb = governor_step(gov, g, mean_now, float((rho ** cfg.material.penalty).mean()))
        vb = min(vb, mean_now + 0.5 * cfg.oc.step_limit)
        new, _ = oc_step(rho, sens, vb, cfg.oc)
        if np.array_equal(new, rho):
            new, _ = oc_step(rho, sens, mean_now - 0.25 * cfg.oc.step_limit, cfg.oc)
        rho = new
        if cfg.symmetry == "central":
            rho = central_symmetrize(rho)
    return rho, kh, log, converged
