"""Device time of one V-cycle (otm_vcycle, graph-captured, 20 per replay) on the
c3 seed design: python tools/vtime.py [n=128] [reps=20].  Env knobs (OTM_*) select
variants; compare runs of this script."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2405_19991_b200 as otm
from paper_2405_19991_b200._dev import Context

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dims = (n, n, n)
rho = otm.init_density(dims, otm.InitPattern("iwp", 0.5, seed=0)).rho
fld = otm.DensityField(dims, rho.copy(), np.zeros(dims))
rho_f = torch.from_numpy(otm.filter_forward(fld, otm.FilterSpec(1.5))).cuda()
ctx = Context(dims)
lib, h = ctx.lib, ctx.h
s = torch.cuda.Stream()
lib.otm_set_stream(h, C.c_void_p(s.cuda_stream))
with torch.cuda.stream(s):
    ctx.check(lib.otm_build(h, C.c_void_p(rho_f.data_ptr())))
    g = torch.Generator(device="cuda").manual_seed(0)
    f = torch.randn(3, n ** 3, device="cuda", dtype=torch.float32, generator=g)
    f -= f.mean(dim=1, keepdim=True)
    z = torch.empty_like(f)
    for _ in range(3):
        ctx.check(lib.otm_vcycle(h, C.c_void_p(f.data_ptr()), C.c_void_p(z.data_ptr())))
s.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=s):
    for _ in range(reps):
        lib.otm_vcycle(h, C.c_void_p(f.data_ptr()), C.c_void_p(z.data_ptr()))
copy = torch.cuda.CUDAGraph()
with torch.cuda.graph(copy, stream=s):
    for _ in range(reps):
        z.copy_(f)
        f.copy_(z)
best = {}
for name, gr in (("vcycle", graph), ("copies", copy)):
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record()
            gr.replay()
            b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / reps * 1e3)
    best[name] = sorted(ts)[len(ts) // 2]
zz = z.double()
print(f"n={n} vcycle+copies {best['vcycle']:.1f} us  copies {best['copies']:.1f} us  "
      f"vcycle ~{best['vcycle'] - best['copies']:.1f} us  |z| {zz.norm().item():.6e}  env "
      + " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("OTM_")))
