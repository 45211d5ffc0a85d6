"""Device plumbing: torch tensors as device memory, the libotm context handle,
error mapping.  No compute happens here.
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_2405_19991_b200 needs a CUDA device (B200, sm_100a); none is visible")
    _lib.load()


def is_tensor(a) -> bool:
    return _torch is not None and isinstance(a, _torch.Tensor) or (
        type(a).__module__.startswith("torch") and hasattr(a, "data_ptr"))


def to_device(a, shape=None, dtype="float64"):
    """Return (contiguous CUDA tensor, came_from_numpy)."""
    require_cuda()
    t = torch()
    tdt = t.float64 if dtype == "float64" else t.float32
    if isinstance(a, t.Tensor):
        out = a.to(device="cuda", dtype=tdt).contiguous()
        host = False
    else:
        arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64 if dtype == "float64" else np.float32))
        out = t.from_numpy(arr).to(device="cuda", non_blocking=False)
        host = True
    if shape is not None and tuple(out.shape) != tuple(shape):
        raise ValueError(f"shape {tuple(out.shape)} != expected {tuple(shape)}")
    return out, host


def like_input(t_out, host: bool):
    return t_out.cpu().numpy() if host else t_out


def ptr(t) -> int:
    return t.data_ptr()


class ConvergenceError(RuntimeError):
    """Solve did not reach the requested residual (solver.py:35-40)."""

    def __init__(self, message: str, residual: float):
        super().__init__(message)
        self.residual = residual


class Context:
    """Owns one otm_ctx (a level hierarchy + device workspaces) and its stream."""

    def __init__(self, dims, kappa0=1.0, kappa_min=1e-4, penalty=3.0, radius=1.5, coarse_target=64,
                 direct_limit=40000, **solver):
        require_cuda()
        t = torch()
        self.lib = _lib.load()
        dev = t.cuda.current_device()
        p = _lib.default_params(kappa0=float(kappa0), kappa_min=float(kappa_min), penalty=float(penalty),
                                filter_radius=float(radius), coarse_target=int(coarse_target),
                                direct_limit=int(direct_limit), device=int(dev))
        for k, v in solver.items():
            setattr(p, k, v)
        h = C.c_void_p()
        rc = self.lib.otm_create(C.byref(h), int(dims[0]), int(dims[1]), int(dims[2]), C.byref(p))
        self.h = h
        if rc != _lib.OTM_OK:
            msg = self.lib.otm_last_error(h).decode() if h.value else "otm_create failed"
            if h.value:
                self.lib.otm_destroy(h)
            self.h = C.c_void_p()
            raise (ValueError if rc == _lib.OTM_EINVAL else RuntimeError)(msg)
        self.dims = tuple(int(d) for d in dims)
        self.n = int(np.prod(self.dims))
        self.device = dev
        self._fin = weakref.finalize(self, self.lib.otm_destroy, h)
        # the library works on its own (non-default, graph-capturable) stream; calls are
        # ordered against torch's current stream with stream waits, not host syncs
        self.stream = t.cuda.Stream(device=dev)
        self.check(self.lib.otm_set_stream(h, C.c_void_p(self.stream.cuda_stream)))
        self.version = 0          # bumped on every solve (invalidates cached results)

    # ------------------------------------------------------------------
    def check(self, rc, residual=None):
        if rc == _lib.OTM_OK:
            return
        msg = self.lib.otm_last_error(self.h).decode()
        if rc == _lib.OTM_EINVAL:
            raise ValueError(msg)
        if rc == _lib.OTM_ENOCONV:
            raise ConvergenceError(msg, float(residual if residual is not None else float("nan")))
        raise RuntimeError(msg)

    def call(self, name, *args):
        cur = torch().cuda.current_stream()
        self.stream.wait_stream(cur)
        rc = getattr(self.lib, name)(self.h, *args)
        cur.wait_stream(self.stream)
        self.check(rc)
        return rc

    def sync(self):
        torch().cuda.synchronize()

    def levels(self):
        out = []
        nl = self.lib.otm_num_levels(self.h)
        for l in range(nl):
            dims = (C.c_int * 3)()
            sc = (C.c_double * 3)()
            self.lib.otm_level_info(self.h, l, dims, sc)
            out.append((tuple(dims), tuple(sc)))
        return out

    def empty(self, *shape):
        return torch().empty(*shape, dtype=torch().float64, device="cuda")


_CACHE: dict = {}


def shared_context(dims, radius=1.5, kappa0=1.0, kappa_min=1e-4, penalty=3.0):
    """A cached context for stateless entry points (filter, symmetry, OC update)."""
    require_cuda()
    key = (tuple(int(d) for d in dims), float(radius), float(kappa0), float(kappa_min), float(penalty),
           torch().cuda.current_device())
    ctx = _CACHE.get(key)
    if ctx is None:
        if len(_CACHE) > 8:
            _CACHE.clear()
        ctx = Context(dims, kappa0=kappa0, kappa_min=kappa_min, penalty=penalty, radius=radius)
        _CACHE[key] = ctx
    return ctx
