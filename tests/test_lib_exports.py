"""CPU-side checks of the drop-in boundary: the sm_100a library builds, loads, exports
every symbol include/fsk.h declares, carries sm_100a SASS, and refuses to run without
an sm_100 device (no CPU fallback). No compute calls are made here."""
import ctypes
import os
import re
import subprocess

import pytest
import torch

from paper_2211_15601_b200 import _lib
from paper_2211_15601_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return _lib.load()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fsk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fsk_\w+)\s*\(", src)))


def test_header_matches_binding_list():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", B.LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (fsk_\w+)", out))
    missing = set(declared_symbols()) - exported
    assert not missing, missing
    for s in declared_symbols():
        assert hasattr(lib, s)


def test_library_carries_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", B.LIB], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_search_kernels_register_budget():
    """The fast pass is sized for FSK_SEARCH_MINB resident CTAs of FSK_SEARCH_BLOCK threads; any local
    memory it needs must stay a few words (no large spills on the hot loop)."""
    out = subprocess.run(["cuobjdump", "-res-usage", B.LIB], capture_output=True, text=True, check=True).stdout
    blocks = out.split("Function ")
    for name in ("13k_search_fast", "18k_search_escalated"):
        k = [b for b in blocks if b.startswith("_ZN3fsk" + name)]
        assert k, name
        stack = int(re.search(r"STACK:(\d+)", k[0]).group(1))
        assert stack <= 32, k[0][:300]


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_device(lib):
    ctx = ctypes.c_void_p()
    rc = lib.fsk_ctx_create(0, ctypes.byref(ctx))
    assert rc == _lib.FSK_ENODEV
    assert b"no CPU fallback" in lib.fsk_last_error() or b"no CUDA device" in lib.fsk_last_error()
    from paper_2211_15601_b200.deformer import Deformer, FskError
    with pytest.raises(FskError):
        Deformer(0)


def test_search_defaults_match_reference(lib):
    d = _lib.GridDesc(4, 4, 4, 2, (ctypes.c_double * 3)(0, 0, 0), (ctypes.c_double * 3)(3, 4, 0))
    o = lib.fsk_search_opts_defaults(ctypes.byref(d))
    # SearchOptions::defaults_for (correspondence.cpp:10-17) with diag = 5
    assert o.max_iters == 50
    for got, want in ((o.conv_eps, 5e-5), (o.div_eps, 2.5), (o.dedup_dist, 0.05)):
        assert abs(got - want) <= 1e-15 * want  # float64 bbox (geometry.hpp:14-39)
