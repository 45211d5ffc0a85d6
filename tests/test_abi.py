"""CPU-only checks of the C ABI: the library loads and exports every symbol that
include/*.h (otm.h, otm_slab.h) declares, and the ctypes table covers them (no
device calls)."""

import ctypes
import os
import re

import pytest

from otm_testutil import ROOT

HEADERS = [os.path.join(ROOT, "include", h) for h in ("otm.h", "otm_slab.h")]
LIB = os.path.join(ROOT, "paper_2405_19991_b200", "libotm.so")


def declared():
    text = "\n".join(open(h).read() for h in HEADERS)
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(otm_[A-Za-z0-9_]+)\s*\(", text)))


def test_header_declares_api():
    names = declared()
    for must in ("otm_create", "otm_solve", "otm_tensor", "otm_sensitivity", "otm_filter", "otm_oc_update",
                 "otm_run_step", "otm_run_update", "otm_governor_update", "otm_vcycle", "otm_slab_stencil",
                 "otm_slab_res64", "otm_slab_restrict", "otm_slab_prolong"):
        assert must in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="libotm.so not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


@pytest.mark.skipif(not os.path.exists(LIB), reason="libotm.so not built")
def test_ctypes_table_matches_header():
    from paper_2405_19991_b200 import _lib
    assert set(_lib.EXPORTED) == set(declared())
    _lib.load()


@pytest.mark.skipif(not os.path.exists(LIB), reason="libotm.so not built")
def test_host_scalar_entry_points_without_gpu():
    """Pure-host C functions (no device work): objective and governor."""
    from paper_2405_19991_b200 import _lib
    import numpy as np
    from oracle import otm_oracle as O
    lib = _lib.load()
    t = [0.3, 0.2, float("nan"), 0.1, 0.02, 0.05]
    k = [0.25, 0.22, 0.4, 0.08, 0.01, 0.0]
    for kind, name in ((0, "mse"), (1, "rel"), (2, "l1")):
        g = ctypes.c_double()
        dG = (ctypes.c_double * 6)()
        assert lib.otm_objective(kind, _lib.doubles(t), _lib.doubles(k), ctypes.byref(g), dG) == 0
        gO, dGO = O.objective(name, t, k)
        assert abs(g.value - gO) <= 1e-15 * max(1.0, gO)
        assert np.allclose(dG[:], dGO, rtol=0, atol=1e-15)
    st = _lib.GovernorC()
    lib.otm_default_governor(ctypes.byref(st))
    gs = O.Governor()
    for gval, mr, mrp in ((5e-5, 0.5, 0.4), (2e-4, 0.45, 0.3), (2.01e-4, 0.44, 0.3), (1e-5, 0.42, 0.3)):
        v = lib.otm_governor_update(ctypes.byref(st), gval, mr, mrp)
        vO = O.governor_step(gs, gval, mr, mrp)
        assert v == vO and st.df == gs.df and st.count == gs.count
