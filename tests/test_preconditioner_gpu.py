"""The MG-PCG preconditioner (one V-cycle, solver.py:326-338 with the damped-Jacobi
smoother) through the C ABI entry point otm_vcycle, on the fast-path level kernels
(k10 level stencils, single-launch 8^3 bottom).  Size-independent properties the
PCG relies on, at BASELINE sizes:

  * symmetry:   <V a, b> = <a, V b>      (fp32 arithmetic: 2e-5 relative)
  * positivity: <V a, a> > 0 on mean-free fields
  * the kernel variants (V-cycle bottom on/off, stored/rebuilt z0, 16-CTA cluster
    tail) are the same linear operator up to fp32 rounding (2e-5 relative)
"""

import ctypes as C

import numpy as np
import pytest

from otm_testutil import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


def _context(dims, seed=0):
    import torch

    import paper_2405_19991_b200 as otm
    from paper_2405_19991_b200._dev import Context

    rng = np.random.default_rng(seed)
    rho = otm.init_density(dims, otm.InitPattern("iwp", 0.5, seed=0)).rho
    rho = np.clip(rho + 0.3 * rng.uniform(-1, 1, dims), 0.001, 1.0)      # contrast + roughness
    fld = otm.DensityField(dims, rho, np.zeros(dims))
    rho_f = torch.from_numpy(otm.filter_forward(fld, otm.FilterSpec(1.5))).cuda()
    ctx = Context(dims)
    ctx.call("otm_build", C.c_void_p(rho_f.data_ptr()))
    return ctx


def _vcycle(ctx, f):
    import torch
    z = torch.empty_like(f)
    ctx.call("otm_vcycle", C.c_void_p(f.data_ptr()), C.c_void_p(z.data_ptr()))
    torch.cuda.synchronize()
    return z


def _fields(n, seed):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn(3, n, device="cuda", dtype=torch.float32, generator=g)
    return (a - a.mean(dim=1, keepdim=True)).contiguous()


@pytest.mark.parametrize("dims", [(64, 64, 64), (128, 128, 128)])
def test_vcycle_symmetric_positive(dims):
    n = int(np.prod(dims))
    ctx = _context(dims)
    a, b = _fields(n, 1), _fields(n, 2)
    va, vb = _vcycle(ctx, a).double(), _vcycle(ctx, b).double()
    a, b = a.double(), b.double()
    for c in range(3):
        lhs = float((va[c] * b[c]).sum())
        rhs = float((a[c] * vb[c]).sum())
        scale = float(va[c].norm() * b[c].norm())
        assert abs(lhs - rhs) <= 2e-5 * scale, (c, lhs, rhs)
        assert float((va[c] * a[c]).sum()) > 0.0


@pytest.mark.parametrize("env", [{"OTM_VBOT": "0"}, {"OTM_VBOT": "16"}])
def test_vcycle_variants_same_operator(env, monkeypatch):
    dims = (128, 128, 128)
    n = int(np.prod(dims))
    a = _fields(n, 3)
    ref = _vcycle(_context(dims), a).double()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    alt = _vcycle(_context(dims), a).double()
    for c in range(3):
        assert float((alt[c] - ref[c]).norm()) <= 2e-5 * float(ref[c].norm())
