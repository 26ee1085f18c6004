"""CPU checks of the C ABI boundary: the library loads and exports every symbol the headers
declare; host-only entry points validate their arguments.  No CUDA call is made here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("moepic.h", "moepic_hostsim.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(moepic_[a-z_]+)\s*\(", src))
    return names


def test_headers_declare_the_boundary():
    names = _declared()
    for core in ("moepic_configure", "moepic_layer_forward", "moepic_predict_prefetch", "moepic_create",
                 "moepic_destroy", "moepic_load_expert", "moepic_load_router"):
        assert core in names


def test_library_exports_every_declared_symbol():
    from paper_2509_08342_b200 import build
    lib_path = build.build()
    lib = ctypes.CDLL(lib_path)
    missing = [n for n in sorted(_declared()) if not hasattr(lib, n)]
    assert not missing, missing
    from paper_2509_08342_b200 import _moepic
    assert set(_moepic.EXPORTED) <= _declared()


def test_arena_bytes_and_desc_validation():
    from paper_2509_08342_b200 import api, _moepic as M
    n = ctypes.c_size_t()
    d = api.model_desc(32, 8, 2, 4096, 14336, max_batch=1, v_e_max=128, L_host=2)
    assert M.moepic_arena_bytes(ctypes.byref(d), ctypes.byref(n)) == M.OK
    # slot pool of 128 experts (45 GB) + 2 ping-pong halves of 4 experts
    assert n.value > 128 * 352321536 + 2 * 4 * 352321536
    # tensor parallel along I: the arena holds the local slice of I / tp_size rows per expert
    nt = ctypes.c_size_t()
    dt = api.model_desc(32, 8, 2, 4096, 14336, max_batch=1, v_e_max=128, L_host=2, tp_rank=1, tp_size=4)
    assert M.moepic_arena_bytes(ctypes.byref(dt), ctypes.byref(nt)) == M.OK
    assert 128 * 352321536 // 4 < nt.value < n.value // 3
    for bad in (dict(K=8), dict(d=4100), dict(I=1000), dict(max_batch=8192), dict(L_host=40),
                dict(tp_size=0), dict(tp_rank=2, tp_size=2), dict(tp_size=3),
                dict(tp_size=2, ep_size=2), dict(I=14336 + 64, tp_size=2),
                dict(max_batch=64, I=14336 + 32, row_granule=32)):   # prefill K tiles need 64-row granules
        kw = dict(L=32, N=8, K=2, d=4096, I=14336, max_batch=1, v_e_max=128, L_host=2)
        kw.update(bad)
        if "I" in bad and "tp_size" in bad:   # I = 14400 = 225 granules: odd, so no even split
            kw["row_granule"] = 64
        d = api.model_desc(**kw)
        assert M.moepic_arena_bytes(ctypes.byref(d), ctypes.byref(n)) == M.EINVAL


def test_no_cpu_fallback_without_library(tmp_path, monkeypatch):
    """The binding refuses to import when libmoepic.so is absent (no silent CPU path)."""
    import importlib.util
    import shutil
    pkg = tmp_path / "pkg"
    pkg.mkdir()
    shutil.copy(os.path.join(ROOT, "paper_2509_08342_b200", "_moepic.py"), pkg / "_moepic.py")
    spec = importlib.util.spec_from_file_location("pkg._moepic", pkg / "_moepic.py")
    mod = importlib.util.module_from_spec(spec)
    with pytest.raises(ImportError):
        spec.loader.exec_module(mod)
