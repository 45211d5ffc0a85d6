"""Design loop: OC updates under the adaptive volume bound (reference: optimize.py).

``run_optimization`` keeps the density, the corrective fields and every
per-element array on the device and advances through ``otm_run_step`` (one C
call per iteration: filter+SIMP, hierarchy, batched MG-PCG, tensor, objective,
sensitivities, adjoint filter, governor, OC multiplier search).  The same
building blocks are exposed one by one with the reference's names.
"""

from __future__ import annotations

import ctypes as C
import math
import threading
import warnings
from dataclasses import dataclass, field as dc_field
from enum import Enum
from typing import Callable, Optional

import numpy as np

from . import _dev, _lib
from .element import MaterialParams
from .field import DensityField, FilterSpec, InitPattern, init_density
from .homogenize import ConductivityTensor, HomogenizationResult
from .objective import KIND_CODE, ObjectiveSpec, feasibility_check


class Model(str, Enum):
    """optimize.py:29-35."""
    ADAPTIVE_OC = "oc"
    MIN_VOLUME_MMA = "mma"
    FIXED_VOLUME_OC = "fixed"


@dataclass
class GovernorState:
    """Adaptive volume ceiling (optimize.py:38-54)."""
    vstar: float = 1.0
    df: float = 1.0
    gap: float = 0.0
    count: int = 0
    bound: float = 1e-4
    iter: int = 0
    g_prev: float = 1.0
    reduced: bool = False

    @property
    def current_decrease(self) -> float:
        return self.gap * self.df if self.reduced else float("inf")

    def _to_c(self):
        return _lib.GovernorC(self.vstar, self.df, self.gap, self.count, self.bound, self.iter, self.g_prev,
                              int(self.reduced))

    def _from_c(self, g):
        self.vstar, self.df, self.gap, self.count = g.vstar, g.df, g.gap, g.count
        self.bound, self.iter, self.g_prev, self.reduced = g.bound, g.iter, g.g_prev, bool(g.reduced)


def _means(rho, penalty):
    t, _ = _dev.to_device(rho)
    ctx = _dev.shared_context(tuple(t.shape))
    out = (C.c_double * 2)()
    ctx.call("otm_means", _dev.ptr(t), float(penalty), out)
    return out[0], out[1]


def governor_update(state: GovernorState, g_now: float, rho, penalty: float) -> float:
    """Algorithm 1 (optimize.py:57-86): device means, host scalar logic in libotm."""
    mean_rho, mean_rho_p = _means(rho, penalty)
    c = state._to_c()
    v = _lib.load().otm_governor_update(C.byref(c), float(g_now), mean_rho, mean_rho_p)
    state._from_c(c)
    return v


@dataclass
class OCParams:
    """optimize.py:89-111."""
    min_density: float = 0.001
    step_limit: float = 0.02
    damp: float = 0.5
    bisection_tol: float = 1e-5

    def __post_init__(self):
        if not (0.0 <= self.min_density < 1.0):
            raise ValueError(f"min_density must be in [0, 1), got {self.min_density}")
        if not (0.0 < self.step_limit <= 1.0):
            raise ValueError(f"step_limit must be in (0, 1], got {self.step_limit}")
        if not (0.0 < self.damp <= 1.0):
            raise ValueError(f"damp must be in (0, 1], got {self.damp}")

    def _to_c(self):
        return _lib.OCParamsC(self.min_density, self.step_limit, self.damp, self.bisection_tol)


EPS_ASCENT = 1e-10


def oc_update(rho, sens, vol_bound: float, params: OCParams):
    """Move-limited OC step with the multiplier bisected on the device (optimize.py:114-160).

    Returns ``(rho_new, {"lam", "active"})``."""
    shape_r = tuple(rho.shape)
    if tuple(sens.shape) != shape_r:
        raise ValueError(f"sensitivity shape {tuple(sens.shape)} != density shape {shape_r}")
    r, host = _dev.to_device(rho)
    s, _ = _dev.to_device(sens)
    ctx = _dev.shared_context(shape_r)
    out = ctx.empty(*shape_r)
    lam = C.c_double(0.0)
    active = C.c_int(0)
    changed = C.c_int(0)
    ctx.call("otm_oc_update", _dev.ptr(r), _dev.ptr(s), float(vol_bound), C.byref(params._to_c()),
             _dev.ptr(out), C.byref(lam), C.byref(active), C.byref(changed))
    return _dev.like_input(out, host), {"lam": float(lam.value), "active": bool(active.value)}


@dataclass
class RunConfig:
    """optimize.py:171-219 (same fields, same validation)."""
    dims: tuple
    target: ObjectiveSpec
    material: MaterialParams = dc_field(default_factory=MaterialParams)
    filter: FilterSpec = dc_field(default_factory=FilterSpec)
    init: InitPattern = dc_field(default_factory=InitPattern)
    init_field: Optional[np.ndarray] = None
    model: Model = Model.ADAPTIVE_OC
    oc: OCParams = dc_field(default_factory=OCParams)
    max_iter: int = 500
    conv_threshold: float = 1e-4
    symmetry: str = "none"
    solver_tol: float = 1e-6
    max_vcycles: int = 200
    governor_bound: float = 1e-4
    volume_bound: Optional[float] = None
    epsilon: float = 1e-4
    mma_move: float = 0.1
    sens_smoothing: bool = False
    dtype: str = "float64"

    def __post_init__(self):
        self.dims = tuple(int(n) for n in self.dims)
        if self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")
        if self.symmetry not in ("none", "central"):
            raise ValueError(f"symmetry must be 'none' or 'central', got {self.symmetry!r}")
        self.model = Model(self.model)
        if self.model is Model.FIXED_VOLUME_OC and self.volume_bound is None:
            raise ValueError("fixed-volume model needs volume_bound")
        if self.model is Model.MIN_VOLUME_MMA and int(np.prod(self.dims)) > 64 ** 3:
            raise ValueError("the MMA path is capped at 64^3 variables; larger grids lose "
                             "volume-gradient precision and exhaust memory, use model 'oc'")
        if self.init_field is not None:
            if hasattr(self.init_field, "data_ptr"):
                arr = self.init_field
                if tuple(arr.shape) != self.dims:
                    raise ValueError(f"init_field shape {tuple(arr.shape)} != dims {self.dims}")
                if float(arr.min()) < 0.0 or float(arr.max()) > 1.0:
                    raise ValueError("init_field densities must lie in [0, 1]")
            else:
                arr = np.asarray(self.init_field, dtype=np.float64)
                if arr.shape != self.dims:
                    raise ValueError(f"init_field shape {arr.shape} != dims {self.dims}")
                if arr.min() < 0.0 or arr.max() > 1.0:
                    raise ValueError("init_field densities must lie in [0, 1]")
                self.init_field = arr


@dataclass
class IterationRecord:
    iter: int
    g: float
    volfrac: float
    volfrac_filtered: float
    vstar: float
    vcycles: int
    ms: float


@dataclass
class OptimizationResult:
    field: DensityField
    kappa: ConductivityTensor
    log: list
    converged: bool
    iterations: int
    config: RunConfig


class OptimizationAborted(RuntimeError):
    """Solver failure mid-run; carries the partial result (optimize.py:243-248)."""

    def __init__(self, message: str, partial: OptimizationResult):
        super().__init__(message)
        self.partial = partial


def _run_config_c(cfg: RunConfig) -> _lib.RunConfigC:
    c = _lib.RunConfigC()
    _lib.load().otm_default_run_config(C.byref(c))
    for i, v in enumerate(cfg.target.target.vec):
        c.target[i] = float(v)
    c.objective = KIND_CODE[cfg.target.kind]
    c.model = 0 if cfg.model is Model.ADAPTIVE_OC else 2
    c.volume_bound = float(cfg.volume_bound) if cfg.volume_bound is not None else float("nan")
    c.oc = cfg.oc._to_c()
    c.max_iter = int(cfg.max_iter)
    c.conv_threshold = float(cfg.conv_threshold)
    c.symmetry = 1 if cfg.symmetry == "central" else 0
    c.solver_tol = float(cfg.solver_tol)
    c.max_vcycles = int(cfg.max_vcycles)
    c.governor_bound = float(cfg.governor_bound)
    return c


def _check_supported(config: RunConfig):
    if config.model is Model.MIN_VOLUME_MMA:
        raise NotImplementedError("model 'mma' (minimum-volume MMA) is outside the B200 hot path")
    if config.sens_smoothing:
        raise NotImplementedError("sensitivity smoothing is off in the reference hot path and not ported")
    if config.filter.kernel is not None:
        raise NotImplementedError("custom filter kernels are not supported on the device path")


class DesignRun:
    """Device-resident state of one run; ``step()`` advances one iteration."""

    def __init__(self, config: RunConfig, hier=None):
        _check_supported(config)
        self.config = config
        from .solver import GridHierarchy
        mp = config.material
        self.hier = hier or GridHierarchy(config.dims, material=mp, filter_radius=config.filter.radius)
        self.hier.set_material(mp)
        t = _dev.torch()
        if config.init_field is not None:
            rho0, _ = _dev.to_device(config.init_field, shape=config.dims)
            rho0 = rho0.clone()
        else:
            rho0, _ = _dev.to_device(init_density(config.dims, config.init).rho)
        # the density lives in one buffer per hierarchy, so the captured iteration graph
        # (which records its address) is reused by every run on this grid
        buf = getattr(self.hier, "_design_rho", None)
        if buf is None or tuple(buf.shape) != tuple(rho0.shape):
            buf = t.empty_like(rho0)
            self.hier._design_rho = buf
        buf.copy_(rho0)
        self.rho = buf
        if config.symmetry == "central":
            self.hier.ctx.call("otm_symmetrize", _dev.ptr(self.rho))
        self.rho_f = t.empty_like(self.rho)
        self.sens = t.empty_like(self.rho)
        self.cc = _run_config_c(config)
        self.st = _lib.RunStateC()
        _lib.load().otm_run_init(C.byref(self.st), C.byref(self.cc))
        self.log: list[IterationRecord] = []
        self.kappa = None

    @property
    def finished(self) -> bool:
        return bool(self.st.finished)

    def evaluate(self):
        """Evaluation half of an iteration (optimize.py:288-345)."""
        rec = _lib.IterRecordC()
        ctx = self.hier.ctx
        cur = _dev.torch().cuda.current_stream()
        ctx.stream.wait_stream(cur)
        rc = ctx.lib.otm_run_step(ctx.h, C.byref(self.cc), C.byref(self.st), _dev.ptr(self.rho),
                                  _dev.ptr(self.rho_f), _dev.ptr(self.sens), C.byref(rec))
        cur.wait_stream(ctx.stream)
        ctx.version += 1
        if rc != _lib.OTM_OK:
            return rc, None
        r = IterationRecord(rec.iter, rec.g, rec.volfrac, rec.volfrac_filtered, rec.vstar, rec.vcycles, rec.ms)
        self.log.append(r)
        self.kappa = ConductivityTensor(np.array(rec.kappa[:]))
        return rc, r

    def update(self):
        """Update half (optimize.py:347-379): governor + OC step, in place."""
        ctx = self.hier.ctx
        cur = _dev.torch().cuda.current_stream()
        ctx.stream.wait_stream(cur)
        rc = ctx.lib.otm_run_update(ctx.h, C.byref(self.cc), C.byref(self.st), _dev.ptr(self.rho))
        cur.wait_stream(ctx.stream)
        ctx.check(rc)

    def step(self):
        rc, rec = self.evaluate()
        if rc == _lib.OTM_OK and not self.finished:
            self.update()
        return rc, rec

    def run_batch(self, max_iters: int, batch: int = 16):
        """Up to ``max_iters`` whole iterations (evaluate + update) as device-resident
        graph launches (otm_run_batch), one host synchronisation per ``batch``.
        Returns (rc, records); rc == OTM_ESTATE means the graph path is unavailable
        and the caller should step() instead."""
        ctx = self.hier.ctx
        recs = (_lib.IterRecordC * int(max_iters))()
        n = C.c_int(0)
        cur = _dev.torch().cuda.current_stream()
        ctx.stream.wait_stream(cur)
        rc = ctx.lib.otm_run_batch(ctx.h, C.byref(self.cc), C.byref(self.st), _dev.ptr(self.rho), int(max_iters),
                                   int(batch), recs, C.byref(n))
        cur.wait_stream(ctx.stream)
        ctx.version += 1
        out = []
        for k in range(n.value):
            r = recs[k]
            rec = IterationRecord(r.iter, r.g, r.volfrac, r.volfrac_filtered, r.vstar, r.vcycles, r.ms)
            self.log.append(rec)
            out.append(rec)
            self.kappa = ConductivityTensor(np.array(r.kappa[:]))
        return rc, out

    def run(self, batch: int = 16):
        """Advance to the end of the run: the graph path when available, else step()."""
        while not self.finished:
            rc, _ = self.run_batch(self.config.max_iter, batch)
            if rc == _lib.OTM_ESTATE and not self.finished:
                rc, _ = self.step()
                while rc == _lib.OTM_OK and not self.finished:
                    rc, _ = self.step()
            if rc != _lib.OTM_OK:
                return rc
        return _lib.OTM_OK

    def error(self) -> str:
        return self.hier.ctx.lib.otm_last_error(self.hier.ctx.h).decode()


_HIER_CACHE: dict = {}          # the main thread's; every other host thread has its own
_TLS = threading.local()


def _hier_cache() -> dict:
    """Per host thread: runs issued from several threads at once (structures designed
    concurrently on one GPU, each on its own hierarchy and stream) never share one."""
    if threading.current_thread() is threading.main_thread():
        return _HIER_CACHE
    cache = getattr(_TLS, "cache", None)
    if cache is None:
        cache = _TLS.cache = {}
    return cache


def _cached_hierarchy(config: RunConfig):
    """Reuse the device hierarchy (buffers, captured graphs) across runs of the same grid.

    A run never depends on what a previous run left in it: otm_run_init starts cold
    (T zeroed on the first evaluation) and every per-iteration buffer is rewritten."""
    from .solver import GridHierarchy
    mp = config.material
    key = (tuple(int(d) for d in config.dims), float(mp.kappa0), float(mp.kappa_min), float(mp.penalty),
           float(config.filter.radius), _dev.torch().cuda.current_device())
    cache = _hier_cache()
    h = cache.get(key)
    if h is None:
        cache.clear()                  # one grid at a time per thread: 512^3 needs ~20 GB
        h = GridHierarchy(config.dims, material=mp, filter_radius=config.filter.radius)
        cache[key] = h
    return h


def run_optimization(config: RunConfig, callback: Optional[Callable] = None,
                     device_result: bool = False) -> OptimizationResult:
    """The full design loop (optimize.py:257-379) on the device.

    The returned field is numpy (as in the reference) unless ``device_result`` or the
    run was seeded from a device tensor.  ``callback(it, fld, result, g)`` receives,
    as in the reference (optimize.py:324-325), the live density field and a
    ``HomogenizationResult`` of this iteration: numpy arrays (``fld.rho``,
    ``result.T_fields``, ``result.rho_filtered``) for host runs, device tensors for
    device runs; ``tensor_sensitivity(result, dG)`` works on it."""
    report = feasibility_check(config.target.target)
    if not report.feasible:
        warnings.warn(f"target tensor is not positive definite (leading minor {report.violated_minor} "
                      "fails); optimization may not reach it", RuntimeWarning)
    _check_supported(config)
    run = DesignRun(config, hier=_cached_hierarchy(config))
    on_device = device_result or hasattr(config.init_field, "data_ptr")
    host_fld = None

    def result(converged):
        rho = run.rho.clone() if on_device else run.rho.cpu().numpy()
        fld = DensityField(config.dims, rho, rho * 0)
        kap = run.kappa if run.kappa is not None else ConductivityTensor(np.full(6, np.nan))
        return OptimizationResult(field=fld, kappa=kap, log=run.log, converged=converged,
                                  iterations=len(run.log), config=config)

    if callback is None:
        # no per-iteration host work: whole iterations as device-resident graph launches
        rc = run.run()
        if rc == _lib.OTM_ENOCONV:
            raise OptimizationAborted(run.error(), result(False))
        if rc != _lib.OTM_OK:
            run.hier.ctx.check(rc)
        return result(bool(run.st.converged))
    while not run.finished:
        rc, rec = run.evaluate()
        if rc == _lib.OTM_ENOCONV:
            raise OptimizationAborted(run.error(), result(False))
        if rc != _lib.OTM_OK:
            run.hier.ctx.check(rc)
        if callback is not None:
            h = run.hier
            T = h.ctx.empty(3, *config.dims)
            h.ctx.call("otm_get_T", _dev.ptr(T))
            if on_device:
                fld = DensityField(config.dims, run.rho, run.sens)
                res = HomogenizationResult(tensor=run.kappa, T_fields=[T[i] for i in range(3)],
                                           rho_filtered=run.rho_f.clone(), params=config.material,
                                           vcycles=rec.vcycles, _hier=h, _version=h.ctx.version)
            else:
                # one DensityField mutated in place across iterations, as the reference's
                # fld; its grad holds the (symmetrised) sensitivity only under central
                # symmetry (optimize.py:308-311)
                if host_fld is None:
                    host_fld = DensityField(config.dims, run.rho.cpu().numpy(), np.zeros(config.dims))
                else:
                    host_fld.rho[...] = run.rho.cpu().numpy()
                if config.symmetry == "central":
                    host_fld.grad[...] = run.sens.cpu().numpy()
                fld = host_fld
                Th = T.cpu().numpy()
                res = HomogenizationResult(tensor=run.kappa, T_fields=[Th[i] for i in range(3)],
                                           rho_filtered=run.rho_f.cpu().numpy(), params=config.material,
                                           vcycles=rec.vcycles, _hier=h, _version=h.ctx.version)
            callback(rec.iter, fld, res, rec.g)
        if not run.finished:
            run.update()
    return result(bool(run.st.converged))
