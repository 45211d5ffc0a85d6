#!/usr/bin/env python
"""Benchmark: seconds per 128^3 anisotropic structure (BASELINE config 3) on B200.

A "step" is one complete structure: 500 OC iterations of the adaptive-volume
loop (``conv_threshold=0`` keeps the count fixed, as BASELINE.md asks for "a
fixed 500 iterations") on the 128^3 IWP seed (vf 0.5), target
[0.3,0.2,0.1,0.1,0.05,0.05] (reference packing k11,k22,k33,k12,k23,k13).

  value  device-timed seconds/structure, density already resident in HBM
  e2e    the same through the public API (run_optimization on a numpy seed,
         H2D of the seed and D2H of the final field inside the timed region);
         first_call_s is the very first call (context + graph setup) on its own
  roofline  dominant kernel class (level-0 MG-PCG stencils) from CUDA events on
         the library stream during the timed region, vs MEASURED_PEAKS.json
  cpu_baseline  the CPU oracle (numpy port of the reference) on the same
         workload: OC iterations 4..6 of one run (warm-started; the reference
         arm's default sample), median x500
  c1_to_convergence / c3_to_convergence  whole runs to the reference's own
         convergence rule (no extrapolation): C1 on both arms, C3 on the GPU
  multi_structure  throughput with 3 structures designed at once on the GPU
         (threads + streams, the gallery's --per-gpu 3); `value` stays the
         one-structure latency

Under ncu (its injection environment) the same kernels run with eager launches from
the host-driven loop, so a launch list can be taken of this command
(profiles/r02zc_bench_launches_c3.md); numbers printed under a profiler are not
bench values.

``--impl reference`` times that CPU port alone (rank 0) on the same metric: one
oracle run, W warm-up iterations (the first is the cold solve from the seed),
then K timed warm-started iterations; value = median x500; plus C1 run to
convergence (unless --no-c1).
Multi-GPU (torchrun): every rank designs its own structure (replicas), value =
max-over-ranks time / (ranks x steps); ``--mode slab`` decomposes ONE structure
into x-slabs over the ranks instead.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TARGET_C3 = [0.3, 0.2, 0.1, 0.1, 0.05, 0.05]
CONFIGS = {
    "c1": dict(dims=(32, 32, 32), target=[0.1, 0.1, 0.1, 0, 0, 0], vf=0.3),
    "c2": dict(dims=(64, 64, 64), target=[0.3, 0.2, 0.1, 0, 0, 0], vf=0.5),
    "c3": dict(dims=(128, 128, 128), target=TARGET_C3, vf=0.5),
    "c4": dict(dims=(256, 256, 256), target=TARGET_C3, vf=0.5),
    "c5": dict(dims=(512, 512, 512), target=[0.1, 0.1, 0.1, 0, 0, 0], vf=0.3),
}
METRIC = "seconds/structure at 128³; MG-PCG stencil GB/s vs B200 HBM peak"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.path = f"/tmp/otm_clocks_{os.getpid()}.csv"
        self.proc = None

    def start(self):
        if os.environ.get("OTM_BENCH_NOCLK"):
            return
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def mark(self):
        """Samples before this call (warm-up) are dropped by stop()."""
        self.skip = 0
        try:
            with open(self.path) as fh:
                self.skip = sum(1 for _ in fh)
        except OSError:
            pass

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for k, line in enumerate(open(self.path)):
            if k < getattr(self, "skip", 0):
                continue
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_config(otm, name, max_iter, conv_threshold, init_field=None):
    c = CONFIGS[name]
    return otm.RunConfig(dims=c["dims"], target=otm.ObjectiveSpec("mse", otm.ConductivityTensor(c["target"])),
                         init=otm.InitPattern("iwp", c["vf"], seed=0), init_field=init_field,
                         max_iter=max_iter, conv_threshold=conv_threshold)


# --------------------------------------------------------------------------- CPU legs
def config_block(name, iters):
    """The `config` object both arms print (identical, so the driver can compare them)."""
    c = CONFIGS[name]
    return {"workload": f"{name} {c['dims']} target {c['target']} (k11,k22,k33,k12,k23,k13), vf {c['vf']}, "
                        f"{iters} OC iterations per structure", "iterations_per_structure": iters,
            "dims": list(c["dims"]), "seed": "iwp (init_density, seed 0)"}


def cpu_iteration_times(name, n_iter):
    """Per-iteration wall times of ONE CPU-oracle run of the workload (iteration 1 is
    the cold solve from the seed, later ones are warm-started as in the reference)."""
    from oracle import otm_oracle as O
    c = CONFIGS[name]
    cfg = O.Run(dims=c["dims"], target=c["target"], init=("iwp", c["vf"], 0), max_iter=n_iter,
                conv_threshold=0.0)
    stamps = [time.perf_counter()]
    O.optimize(cfg, callback=lambda *a: stamps.append(time.perf_counter()))
    return [b - a for a, b in zip(stamps, stamps[1:])]


def multi_structure(otm, torch, name, iters, seed, k=3):
    """Throughput with k independent structures designed at once on this GPU (the
    gallery's `--per-gpu k`): one host thread, hierarchy, CUDA stream and captured
    iteration graph each; device time from the first launch to the last completion
    (events on the default stream bracketing the k runs), against the same k runs
    one after another."""
    import threading
    from paper_2405_19991_b200.optimize import DesignRun
    from paper_2405_19991_b200.solver import GridHierarchy
    cfg = make_config(otm, name, iters, 0.0, init_field=seed)
    hiers = [GridHierarchy(cfg.dims, material=cfg.material, filter_radius=cfg.filter.radius) for _ in range(k)]
    streams = [torch.cuda.Stream() for _ in range(k)]
    logs = [None] * k

    def one(i):
        with torch.cuda.stream(streams[i]):
            run = DesignRun(cfg, hier=hiers[i])
            run.run()
            logs[i] = run.log

    def timed(concurrent):
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        if concurrent:
            th = [threading.Thread(target=one, args=(i,)) for i in range(k)]
            for t in th:
                t.start()
            for t in th:
                t.join()
        else:
            for i in range(k):
                one(i)
        cur = torch.cuda.current_stream()
        for st in streams:
            cur.wait_stream(st)
        ev[1].record()
        ev[1].synchronize()
        return ev[0].elapsed_time(ev[1]) / 1e3

    timed(False)                                   # capture every hierarchy's graphs
    seq = timed(False)
    conc = timed(True)
    same = all(len(lg) == len(logs[0]) and all(a.g == b.g for a, b in zip(lg, logs[0])) for lg in logs)
    del hiers
    return {"value": conc / k, "unit": "s/structure", "one_at_a_time_s": seq / k, "speedup": seq / conc,
            "identical_results": bool(same),
            "note": f"{k} {name} structures at once on one GPU (threads + streams), device time / {k}"}


def cpu_to_convergence(name):
    """The CPU oracle run to the reference's convergence rule: (seconds, iterations, g)."""
    from oracle import otm_oracle as O
    c = CONFIGS[name]
    cfg = O.Run(dims=c["dims"], target=c["target"], init=("iwp", c["vf"], 0), max_iter=500)
    t0 = time.perf_counter()
    rho, kh, log, conv = O.optimize(cfg)
    return time.perf_counter() - t0, len(log), float(log[-1].g), bool(conv)


def run_reference(args):
    world, rank, _ = dist_init()
    if rank != 0:
        return
    times = cpu_iteration_times(args.config, args.warmup + args.steps)
    timed = times[args.warmup:]
    s_iter = statistics.median(timed)
    value = s_iter * args.iters
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "s/structure",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": s_iter * 1e3, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (IWP seed, reference init_density)",
            "config": config_block(args.config, args.iters),
            "step": "one warm-started OC iteration of the CPU oracle (filter, 3 GS-V-cycle solves, tensor, "
                    "sensitivities, adjoint filter, governor, OC) inside one run; value = median x iterations",
            "iteration_s": {"cold_first": round(times[0], 3), "timed": [round(t, 3) for t in timed],
                            "median": round(s_iter, 3), "mean": round(statistics.mean(timed), 3)},
            "cpu_baseline": {"value": value, "unit": "s/structure", "cores": 1, "kind": "port",
                             "sample": f"iterations {args.warmup + 1}..{args.warmup + args.steps} of one oracle run "
                                       f"on {args.config} (warm-started), median x{args.iters}; the cold first "
                                       f"iteration took {times[0]:.1f} s"},
            "e2e": {"value": value, "unit": "s/structure", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not args.no_c1:
        secs, its, g, conv = cpu_to_convergence("c1")
        line["c1_to_convergence"] = {"value": secs, "unit": "s/structure", "iterations": its, "final_g": g,
                                     "converged": conv, "workload": config_block("c1", 500)["workload"]
                                     + " (stops at the reference's convergence rule)"}
    print(json.dumps(line), flush=True)


def traffic_bytes(name):
    """ncu DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch of the
    level-0 stencil class of workload `name`, mean over smooth_res / jacobi / spmv,
    from the newest committed ncu --set full capture of THAT workload
    (profiles/r*_traffic_<name>.json); None without one."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_traffic_{name}.json")))
    if not files:
        return None
    try:
        return json.load(open(files[-1]))["mean_dram_bytes"]
    except (OSError, ValueError, KeyError):
        return None


def beyond_l2(otm, _lib, lib, torch, peak, peak_kind, iters=20):
    """The same level-0 stencil roofline on c4 = 256³, where the three fp32 load-case
    fields (64 MB each) no longer fit the 126 MB L2: one instrumented 20-iteration
    structure from the IWP seed (CUDA events around every level-0 stencil launch).
    Explains `roofline` (128³ is L2-resident and latency-bound); not the headline."""
    import ctypes as C
    from paper_2405_19991_b200.optimize import DesignRun
    try:
        dims = CONFIGS["c4"]["dims"]
        seed = torch.from_numpy(otm.init_density(dims, otm.InitPattern("iwp", CONFIGS["c4"]["vf"], seed=0)).rho).cuda()
        hier = otm.GridHierarchy(dims)
        ctx = hier.ctx

        def structure():
            run = DesignRun(make_config(otm, "c4", iters, 0.0, init_field=seed), hier=hier)
            while not run.finished:
                rc, _ = run.step()
                if rc != _lib.OTM_OK:
                    ctx.check(rc)

        structure()                                  # warm-up (graphs, tensor maps)
        torch.cuda.synchronize()
        lib.otm_profile_reset(ctx.h)
        lib.otm_profile_enable(ctx.h, 1)
        structure()
        torch.cuda.synchronize()
        lib.otm_profile_enable(ctx.h, 0)
        out = {}
        for cls, nm in ((0, "l0_stencil"), (1, "vcycle")):
            ms_t, cnt, byt = C.c_double(), C.c_longlong(), C.c_double()
            lib.otm_profile_read(ctx.h, cls, C.byref(ms_t), C.byref(cnt), C.byref(byt))
            gbs = (byt.value / (ms_t.value * 1e-3) / 1e9) if ms_t.value > 0 else None
            out[nm] = {"ms": ms_t.value, "launches": cnt.value, "gbs": gbs,
                       "frac": (gbs / peak) if gbs else None}
        del hier, ctx
        torch.cuda.empty_cache()
        return {"workload": f"c4 {dims}, {iters} OC iterations from the IWP seed", "bound": "hbm",
                "unit": "GB/s", "peak": peak, "peak_kind": peak_kind,
                "achieved": out["l0_stencil"]["gbs"], "frac": out["l0_stencil"]["frac"], "kernels": out,
                "traffic": traffic_bytes("c4"),
                "traffic_note": "mean ncu DRAM bytes per level-0 stencil launch at 256^3 "
                                "(profiles/r*_traffic_c4.json); algorithmic 44/44/28 B per vertex"}
    except Exception as e:                           # reported, never fatal to the headline line
        return {"error": f"{type(e).__name__}: {e}"}


# --------------------------------------------------------------------------- GPU leg
def run_gpu(args):
    import numpy as np
    import torch

    world, rank, local = dist_init()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2405_19991_b200 as otm
    from paper_2405_19991_b200 import _dev, _lib
    from paper_2405_19991_b200.optimize import DesignRun

    name = args.config
    dims = CONFIGS[name]["dims"]
    n = int(np.prod(dims))
    seed = otm.init_density(dims, otm.InitPattern("iwp", CONFIGS[name]["vf"], seed=0)).rho
    seed_dev = torch.from_numpy(seed).cuda()
    lib = _lib.load()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")   # > 126 MB L2

    hier = otm.GridHierarchy(dims)
    ctx = hier.ctx

    def one_structure():
        cfg = make_config(otm, name, args.iters, 0.0, init_field=seed_dev)
        run = DesignRun(cfg, hier=hier)
        if args.host_loop:
            while not run.finished:
                rc, _ = run.step()
                if rc != _lib.OTM_OK:
                    ctx.check(rc)
        else:
            rc = run.run()                   # device-resident iterations (host path while profiling)
            if rc != _lib.OTM_OK:
                ctx.check(rc)
        return run

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # the clock sampler starts before the warm-up: nvidia-smi's own start-up (NVML
    # init) stalled CUDA API calls of the design loop for up to ~0.3 s when it landed
    # inside a timed step; only the samples taken from the timed region on are kept
    clocks = Clocks(local)
    clocks.start()
    for _ in range(args.warmup):
        one_structure()
    barrier()
    # ---- timed region (device events on the library stream, no instrumentation) ----
    launches0 = lib.otm_launch_count(ctx.h)
    lib.otm_stats_reset(ctx.h)
    clocks.mark()
    step_ms = []
    iters_done = []
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    total_ms = 0.0
    gc.collect()
    gc.disable()                         # as timeit does: no collector pauses inside timed steps
    for _ in range(args.steps):
        flush.fill_(1.0)                 # evict L2 between steps
        barrier()
        ev[0].record(ctx.stream)
        run = one_structure()
        ev[1].record(ctx.stream)
        ev[1].synchronize()
        ms = ev[0].elapsed_time(ev[1])
        step_ms.append(ms)
        total_ms += ms
        iters_done.append(len(run.log))
    barrier()
    gc.enable()
    clk = clocks.stop()
    launches = lib.otm_launch_count(ctx.h) - launches0
    import ctypes as C
    st = (C.c_longlong * 6)()
    lib.otm_stats(ctx.h, st)
    solver_stats = {"solves": st[0], "fp64_refinements_per_solve": st[1] / max(st[0], 1),
                    "pcg_iterations_per_oc_iteration": st[2] / max(st[0], 1),
                    "vcycles_per_oc_iteration": sum(r.vcycles for r in run.log) / max(len(run.log), 1),
                    "oc_passes_per_update": st[4] / max(st[3], 1), "frozen_retries": st[5]}
    ph = (C.c_double * 4)()
    lib.otm_loop_phases(ctx.h, ph)
    n_it = max(sum(iters_done), 1)
    if ph[0] > 0:
        solver_stats["iteration_phases_us"] = {
            "filter_build_solve": round(ph[0] * 1e3 / n_it, 1), "tensor_objective": round(ph[1] * 1e3 / n_it, 1),
            "sens_filter_oc": round(ph[2] * 1e3 / n_it, 1), "gap": round(ph[3] * 1e3 / n_it, 1),
            "note": "graph path, %globaltimer stamps of the loop-control kernels, mean per OC iteration"}
    # max over ranks
    t_max = total_ms
    if world > 1:
        tt = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_max = float(tt.item())
    value = (t_max / 1e3) / (args.steps * world)
    # ---- kernel classes: CUDA event pairs recorded around every level-0 stencil launch
    # (inside the inner-iteration graph) while one more structure of the same workload
    # runs right after the timed region ----
    import ctypes as C
    lib.otm_profile_reset(ctx.h)
    lib.otm_profile_enable(ctx.h, 0 if args.no_prof else 1)
    flush.fill_(1.0)
    barrier()
    one_structure()
    barrier()
    lib.otm_profile_enable(ctx.h, 0)
    prof = {}
    for cls, nm in ((0, "l0_stencil"), (1, "vcycle"), (2, "res64"), (3, "tensor_sens"), (4, "filter"), (5, "oc")):
        ms_t, cnt, byt = C.c_double(), C.c_longlong(), C.c_double()
        lib.otm_profile_read(ctx.h, cls, C.byref(ms_t), C.byref(cnt), C.byref(byt))
        prof[nm] = {"ms": ms_t.value, "launches": cnt.value, "bytes": byt.value,
                    "gbs": (byt.value / (ms_t.value * 1e-3) / 1e9) if ms_t.value > 0 else None}
    peak, peak_kind = peaks()
    l0 = prof["l0_stencil"]
    achieved = l0["gbs"]
    # ---- e2e through the public API with host buffers ----
    from paper_2405_19991_b200 import optimize as _opt
    e2e_ms = []
    gc.collect()
    gc.disable()
    torch.cuda.synchronize()
    torch_base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    for s in range(4):                                   # run 0: first call (hierarchy + graph setup)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cfg = make_config(otm, name, args.iters, 0.0, init_field=seed)     # numpy seed: H2D inside
        if s == 0 and os.environ.get("OTM_BENCH_PSTATS"):                    # where a slow first call went
            import cProfile
            import pstats
            pr = cProfile.Profile()
            res = pr.runcall(otm.run_optimization, cfg)
            pstats.Stats(pr, stream=sys.stderr).sort_stats("tottime").print_stats(10)
        else:
            res = otm.run_optimization(cfg)                                 # numpy field back: D2H inside
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        assert isinstance(res.field.rho, np.ndarray)
    gc.enable()
    torch_peak = torch.cuda.max_memory_allocated() - torch_base
    lib_bytes = sum(int(lib.otm_device_bytes(h.ctx.h)) for h in _opt._HIER_CACHE.values())
    e2e = statistics.median(e2e_ms[1:]) / 1e3
    if world > 1:
        tt = torch.tensor([e2e], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e = float(tt.item()) / world
    # ---- whole runs to the reference's convergence rule (no fixed count, no extrapolation) ----
    conv = {}
    if world == 1:
        for cname in ([] if args.no_c1 else ["c1"]) + ([name] if name != "c1" else []):
            walls = []
            for _ in range(2):                           # second run: hierarchy cached
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                r = otm.run_optimization(make_config(otm, cname, 500, 1e-4,
                                                     init_field=otm.init_density(
                                                         CONFIGS[cname]["dims"],
                                                         otm.InitPattern("iwp", CONFIGS[cname]["vf"], 0)).rho))
                torch.cuda.synchronize()
                walls.append(time.perf_counter() - t0)
            conv[cname] = {"value": walls[1], "unit": "s/structure", "first_call_s": walls[0],
                           "iterations": r.iterations, "final_g": r.log[-1].g, "converged": r.converged,
                           "final_volfrac": r.field.mean(),
                           "workload": config_block(cname, 500)["workload"]
                           + " (stops at the reference's convergence rule)",
                           "path": "run_optimization (numpy seed in, numpy field out), host wall clock"}
    multi = multi_structure(otm, torch, name, args.iters, seed_dev) if (world == 1 and args.multi > 1) else None
    if multi:
        multi["structures_per_gpu"] = args.multi
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "s/structure", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32",
        "data": "synthetic (IWP seed from init_density, vf 0.5)",
        "config": config_block(name, args.iters),
        "run": {"iterations_per_step": iters_done, "step_ms": [round(x, 2) for x in step_ms],
                "parallelism": f"replicas x{world}",
                "l2": "flushed (256 MB write) before every timed step",
                "solver": "fp64 defect correction + fp32 MG-PCG (damped Jacobi V-cycle), tol 1e-6"},
        "solver_stats": solver_stats,
        "device_memory": {"libotm_bytes": lib_bytes, "torch_peak_bytes": int(torch_peak),
                          "total_mb": round((lib_bytes + torch_peak) / 2**20, 1),
                          "note": "one run_optimization of the workload: the hierarchy context (libotm) + "
                                  "the torch-held fields (density, filtered density, sensitivities)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic_bytes(name),
                     "kernel": "level-0 stencils (smooth_res + jacobi + spmv), 3 load cases fp32",
                     "bytes_per_vertex": "44 (smooth_res, jacobi) / 28 (spmv)", "peak_kind": peak_kind,
                     "measured": "CUDA events on the library stream around every level-0 stencil launch, "
                                 "one instrumented structure of the same workload run right after the timed steps"},
        "kernels": prof,
        "gpu_launches": int(launches),
        "clocks": clk,
        "e2e": {"value": e2e, "unit": "s/structure", "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                "first_call_s": round(e2e_ms[0] / 1e3, 4), "runs_s": [round(x / 1e3, 4) for x in e2e_ms[1:]],
                "path": "run_optimization(RunConfig(init_field=numpy seed)) -> numpy rho; value = median of "
                        "the runs after the first (the first allocates the hierarchy and captures its graphs)"},
    }
    for cname, rec in conv.items():
        line[f"{cname}_to_convergence"] = rec
    if multi:
        line["multi_structure"] = multi
    if args.beyond_l2 and world == 1 and name != "c4":
        line["roofline_beyond_l2"] = beyond_l2(otm, _lib, lib, torch, peak, peak_kind)
    if not args.no_cpu and world == 1:
        # the reference arm's default sample (--warmup 3 --steps 3): iterations 4..6
        t = cpu_iteration_times(name, 6)
        med = statistics.median(t[3:6])
        line["cpu_baseline"] = {"value": med * args.iters, "unit": "s/structure", "cores": 1, "kind": "port",
                                "sample": f"iterations 4..6 of one oracle run on {name} (warm-started; "
                                          f"{', '.join(f'{x:.1f}' for x in t[3:6])} s), median x{args.iters}; "
                                          f"iterations 1..3 took {', '.join(f'{x:.1f}' for x in t[:3])} s"}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()



# --------------------------------------------------------------------------- slab leg
def run_slab(args):
    """--mode slab: ONE structure decomposed into x-slabs over the ranks (strong
    scaling; SlabDesignRun over NCCL, paper_2405_19991_b200/slab.py).  N=1 runs a
    single slab in-process."""
    import numpy as np
    import torch

    world, rank, local = dist_init()
    torch.cuda.set_device(local)
    import paper_2405_19991_b200 as otm
    from paper_2405_19991_b200.slab import CudaSlabBackend, DistComm, LocalComm, SlabDesignRun
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = DistComm()
    else:
        comm = LocalComm(1)
    name = args.config
    dims = CONFIGS[name]["dims"]
    seed = otm.init_density(dims, otm.InitPattern("iwp", CONFIGS[name]["vf"], seed=0)).rho
    nxl = dims[0] // world
    part = torch.from_numpy(np.ascontiguousarray(seed[rank * nxl:(rank + 1) * nxl])).cuda()
    backend = CudaSlabBackend(3 * nxl * dims[1] * dims[2])

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def one_structure():
        cfg = make_config(otm, name, args.iters, 0.0)
        run = SlabDesignRun(cfg, comm, backend, [part])
        while not run.finished:
            run.step()
        return run

    for _ in range(args.warmup):
        one_structure()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    total = 0.0
    iters = []
    for _ in range(args.steps):
        barrier()
        ev[0].record()
        run = one_structure()
        ev[1].record()
        ev[1].synchronize()
        total += ev[0].elapsed_time(ev[1])
        iters.append(len(run.log))
    barrier()
    t_max = total
    if world > 1:
        tt = torch.tensor([total], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_max = float(tt.item())
    value = t_max / 1e3 / args.steps
    # the same workload on ONE GPU through the single-GPU solver (rank 0): the
    # reference point of the strong-scaling efficiency T1 / (N * TN)
    single = None
    if rank == 0 and not args.no_single:
        from paper_2405_19991_b200.optimize import DesignRun
        hier = otm.GridHierarchy(dims)
        seed_dev = torch.from_numpy(seed).cuda()

        def one_single():
            r = DesignRun(make_config(otm, name, args.iters, 0.0, init_field=seed_dev), hier=hier)
            r.run()
            return r

        one_single()
        ts = []
        for _ in range(max(1, args.steps)):
            torch.cuda.synchronize()
            ev[0].record()
            one_single()
            ev[1].record()
            ev[1].synchronize()
            ts.append(ev[0].elapsed_time(ev[1]) / 1e3)
        single = statistics.median(ts)
        del hier
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "s/structure", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic (IWP seed from init_density)",
                "config": {"workload": f"{name} {dims} target {CONFIGS[name]['target']}, {args.iters} OC iterations, "
                                       f"one structure on {world} x-slabs",
                           "mode": "slab", "iterations_per_step": iters,
                           "parallelism": f"x-slabs x{world}, NCCL halos + all-reduce"}}
        if single is not None:
            line["single_gpu"] = {"value": single, "unit": "s/structure",
                                  "path": "the single-GPU solver (iteration graph) on the same workload, rank 0"}
            line["slab_over_single"] = value / single
            line["parallel_efficiency"] = single / (world * value)
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--iters", type=int, default=500, help="OC iterations per structure")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-c1", action="store_true", help="skip the C1 to-convergence legs")
    ap.add_argument("--multi", type=int, default=3,
                    help="structures designed at once for the multi_structure key (<= 1: skip)")
    ap.add_argument("--no-single", action="store_true", help="--mode slab: skip the single-GPU reference time")
    ap.add_argument("--host-loop", action="store_true",
                    help="drive the design loop from the host (otm_run_step/update) instead of the iteration graph")
    ap.add_argument("--no-prof", action="store_true", help="no in-region kernel events")
    ap.add_argument("--no-beyond-l2", dest="beyond_l2", action="store_false",
                    help="skip the 256³ level-0 stencil roofline leg")
    ap.add_argument("--mode", default="replicas", choices=["replicas", "slab"],
                    help="N>1: independent structures per rank (default) or one structure on x-slabs")
    args = ap.parse_args()
    if any(os.environ.get(k) for k in ("NV_NSIGHT_INJECTION_TRANSPORT_TYPE", "NV_TPS_LAUNCH_TOKEN",
                                       "CUDA_INJECTION64_PATH")):
        # under a profiler (ncu's injection environment): kernel nodes of graphs with
        # conditional nodes cannot be profiled one by one, so run the same kernels
        # from the host (eager launches, host-driven design loop); a number printed
        # under a profiler is never a bench value
        for k in ("OTM_NO_ITER_GRAPH", "OTM_NO_LOOP_GRAPH", "OTM_EAGER"):
            os.environ.setdefault(k, "1")
        args.host_loop = True
    if args.impl == "reference":
        run_reference(args)
    elif args.mode == "slab":
        run_slab(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
