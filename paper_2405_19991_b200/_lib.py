"""ctypes binding of libotm.so (the C ABI in include/otm.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or ``make``
in ``csrc/``).  There is no fallback: if the library is missing or no CUDA
device is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OTM_LIB", os.path.join(_HERE, "libotm.so"))

OTM_OK, OTM_EINVAL, OTM_ENOCONV, OTM_ECUDA, OTM_ESTATE = 0, 1, 2, 3, 4

dptr = C.c_void_p


class Params(C.Structure):
    _fields_ = [("kappa0", C.c_double), ("kappa_min", C.c_double), ("penalty", C.c_double),
                ("filter_radius", C.c_double), ("coarse_target", C.c_int), ("direct_limit", C.c_int),
                ("jacobi_omega", C.c_double), ("inner_reduction", C.c_double), ("max_inner", C.c_int),
                ("device", C.c_int)]


class OCParamsC(C.Structure):
    _fields_ = [("min_density", C.c_double), ("step_limit", C.c_double), ("damp", C.c_double),
                ("bisection_tol", C.c_double)]


class GovernorC(C.Structure):
    _fields_ = [("vstar", C.c_double), ("df", C.c_double), ("gap", C.c_double), ("count", C.c_int),
                ("bound", C.c_double), ("iter", C.c_int), ("g_prev", C.c_double), ("reduced", C.c_int)]


class IterRecordC(C.Structure):
    _fields_ = [("iter", C.c_int), ("g", C.c_double), ("volfrac", C.c_double),
                ("volfrac_filtered", C.c_double), ("vstar", C.c_double), ("vcycles", C.c_int),
                ("ms", C.c_double), ("kappa", C.c_double * 6), ("solve_residual", C.c_double * 3)]


class RunConfigC(C.Structure):
    _fields_ = [("target", C.c_double * 6), ("objective", C.c_int), ("model", C.c_int),
                ("volume_bound", C.c_double), ("oc", OCParamsC), ("max_iter", C.c_int),
                ("conv_threshold", C.c_double), ("symmetry", C.c_int), ("solver_tol", C.c_double),
                ("max_vcycles", C.c_int), ("governor_bound", C.c_double)]


class RunStateC(C.Structure):
    _fields_ = [("gov", GovernorC), ("iter", C.c_int), ("plateau", C.c_int), ("have_g_last", C.c_int),
                ("g_last", C.c_double), ("converged", C.c_int), ("finished", C.c_int), ("warm", C.c_int),
                ("g", C.c_double), ("mean_rho", C.c_double), ("mean_rho_p", C.c_double)]


_SIGS = {
    "otm_default_params": (None, [C.POINTER(Params)]),
    "otm_default_oc_params": (None, [C.POINTER(OCParamsC)]),
    "otm_default_run_config": (None, [C.POINTER(RunConfigC)]),
    "otm_default_governor": (None, [C.POINTER(GovernorC)]),
    "otm_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, C.POINTER(Params)]),
    "otm_destroy": (C.c_int, [C.c_void_p]),
    "otm_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "otm_last_error": (C.c_char_p, [C.c_void_p]),
    "otm_version": (C.c_char_p, []),
    "otm_num_levels": (C.c_int, [C.c_void_p]),
    "otm_level_info": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double)]),
    "otm_device_bytes": (C.c_size_t, [C.c_void_p]),
    "otm_set_material": (C.c_int, [C.c_void_p, C.c_double, C.c_double, C.c_double]),
    "otm_filter": (C.c_int, [C.c_void_p, dptr, dptr, C.c_int]),
    "otm_symmetrize": (C.c_int, [C.c_void_p, dptr]),
    "otm_build": (C.c_int, [C.c_void_p, dptr]),
    "otm_build_kappa": (C.c_int, [C.c_void_p, dptr]),
    "otm_apply_K": (C.c_int, [C.c_void_p, dptr, dptr]),
    "otm_macro_load": (C.c_int, [C.c_void_p, C.c_int, dptr]),
    "otm_set_warm": (C.c_int, [C.c_void_p, dptr]),
    "otm_solve": (C.c_int, [C.c_void_p, dptr, C.c_double, C.c_int, C.POINTER(C.c_int),
                            C.POINTER(C.c_double)]),
    "otm_get_T": (C.c_int, [C.c_void_p, dptr]),
    "otm_residual_history": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_int]),
    "otm_level_kappa": (C.c_int, [C.c_void_p, C.c_int, dptr]),
    "otm_level_apply": (C.c_int, [C.c_void_p, C.c_int, dptr, dptr, dptr]),
    "otm_relax_gs8": (C.c_int, [C.c_void_p, C.c_int, dptr, dptr, C.c_int]),
    "otm_restrict": (C.c_int, [C.c_void_p, C.c_int, dptr, dptr]),
    "otm_prolong_correct": (C.c_int, [C.c_void_p, C.c_int, dptr, dptr]),
    "otm_coarse_solve": (C.c_int, [C.c_void_p, dptr, dptr]),
    "otm_tensor": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "otm_pair_energy": (C.c_int, [C.c_void_p, dptr]),
    "otm_elem_diff": (C.c_int, [C.c_void_p, dptr, C.c_int, dptr]),
    "otm_sensitivity": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), dptr]),
    "otm_objective": (C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "otm_means": (C.c_int, [C.c_void_p, dptr, C.c_double, C.POINTER(C.c_double)]),
    "otm_oc_update": (C.c_int, [C.c_void_p, dptr, dptr, C.c_double, C.POINTER(OCParamsC), dptr,
                                C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "otm_governor_update": (C.c_double, [C.POINTER(GovernorC), C.c_double, C.c_double, C.c_double]),
    "otm_run_init": (None, [C.POINTER(RunStateC), C.POINTER(RunConfigC)]),
    "otm_run_step": (C.c_int, [C.c_void_p, C.POINTER(RunConfigC), C.POINTER(RunStateC), dptr, dptr, dptr,
                               C.POINTER(IterRecordC)]),
    "otm_run_update": (C.c_int, [C.c_void_p, C.POINTER(RunConfigC), C.POINTER(RunStateC), dptr]),
    "otm_run_batch": (C.c_int, [C.c_void_p, C.POINTER(RunConfigC), C.POINTER(RunStateC), dptr, C.c_int, C.c_int,
                                C.POINTER(IterRecordC), C.POINTER(C.c_int)]),
    "otm_profile_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "otm_profile_read": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_longlong),
                                   C.POINTER(C.c_double)]),
    "otm_profile_reset": (C.c_int, [C.c_void_p]),
    "otm_launch_count": (C.c_longlong, [C.c_void_p]),
    "otm_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_longlong)]),
    "otm_stats_reset": (C.c_int, [C.c_void_p]),
    "otm_loop_phases": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "otm_vcycle": (C.c_int, [C.c_void_p, dptr, dptr]),
    # include/otm_slab.h: slab-decomposed solve pieces (multi-GPU)
    "otm_slab_create": (C.c_void_p, [C.c_longlong]),
    "otm_slab_destroy": (C.c_int, [C.c_void_p]),
    "otm_slab_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "otm_slab_last_error": (C.c_char_p, [C.c_void_p]),
    "otm_slab_stencil": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double), dptr,
                                   dptr, dptr, dptr, C.c_double, dptr, dptr, C.POINTER(C.c_double)]),
    "otm_slab_stencil_range": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                                         dptr, dptr, dptr, dptr, C.c_double, dptr, dptr, C.c_int, C.c_int,
                                         C.POINTER(C.c_double)]),
    "otm_slab_set_scalar_mode": (C.c_int, [C.c_void_p, C.c_int]),
    "otm_slab_pcg_step": (C.c_int, [C.c_void_p, C.c_int, dptr]),
    "otm_slab_halo_local": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_longlong, C.c_void_p, C.c_int, C.c_void_p,
                                      C.c_int, C.c_void_p, C.c_int]),
    "otm_slab_restrict": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, dptr, dptr]),
    "otm_slab_prolong": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, dptr, dptr]),
    "otm_slab_coarsen": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, dptr, dptr]),
    "otm_slab_dinv": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double), dptr, dptr]),
    "otm_slab_pupd": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, dptr, dptr, C.POINTER(C.c_double)]),
    "otm_slab_upd": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, dptr, dptr, dptr, dptr,
                               C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "otm_slab_load_sums": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double), dptr,
                                     C.POINTER(C.c_double)]),
    "otm_slab_res64": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double), dptr, dptr,
                                 C.POINTER(C.c_double), dptr, C.POINTER(C.c_double)]),
    "otm_slab_tupd": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, dptr, dptr, C.POINTER(C.c_double)]),
    "otm_slab_tensor_sums": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double), dptr, dptr,
                                       C.POINTER(C.c_double)]),
    "otm_slab_filter": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                  C.c_double, C.c_double, dptr, dptr, dptr, C.POINTER(C.c_double)]),
    "otm_slab_sensitivity": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                       C.c_double, dptr, dptr, C.POINTER(C.c_double), dptr]),
    "otm_slab_oc_sums": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, C.POINTER(OCParamsC), dptr,
                                   dptr, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "otm_slab_oc_apply": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, C.POINTER(OCParamsC), dptr,
                                    dptr, C.c_double, dptr, C.POINTER(C.c_double)]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


class LibraryMissing(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load libotm.so once; raise loudly when it was not built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise LibraryMissing(
                f"{path} not found: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        lib = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def default_params(**kw) -> Params:
    p = Params()
    load().otm_default_params(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def default_oc() -> OCParamsC:
    p = OCParamsC()
    load().otm_default_oc_params(C.byref(p))
    return p


def doubles(vals):
    arr = (C.c_double * len(vals))(*[float(v) for v in vals])
    return arr
