"""The C-ABI library loads without a GPU and exports every function that
include/*.h declares (no compute calls: those need a device)."""
import ctypes
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"\b(yy_[a-z_]+)\s*\(", txt):
            names.add(m.group(1))
    return names


def test_headers_declare_the_core_calls():
    d = _declared()
    for n in ("yy_create", "yy_set_fields", "yy_step", "yy_get_fields", "yy_destroy"):
        assert n in d


def test_library_exports_every_declared_symbol():
    import paper_1905_02300_b200 as pkg
    if not os.path.exists(pkg.lib_path()):
        import __graft_entry__
        __graft_entry__.build()
    lib = ctypes.CDLL(pkg.lib_path())
    missing = [n for n in sorted(_declared()) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(pkg.yy.EXPORTS) <= _declared()


def test_binding_refuses_without_library(tmp_path, monkeypatch):
    import paper_1905_02300_b200.yy as yy
    monkeypatch.setattr(yy, "_lib", None)
    monkeypatch.setattr(yy, "_HERE", str(tmp_path))
    try:
        yy.load_library()
    except yy.YYError:
        return
    raise AssertionError("binding must fail loudly when libyy.so is missing")


def test_allocator_hook_host_logic():
    """yy_set_allocator: process default only (ctx = NULL), alloc / free in pairs."""
    import paper_1905_02300_b200 as pkg
    from paper_1905_02300_b200.yy import ALLOC_FN, FREE_FN
    L = pkg.load_library()
    assert L.yy_set_allocator(None, ALLOC_FN(), FREE_FN(), None) == 0            # reset: cudaMalloc
    half = ALLOC_FN(lambda n, u: 0)
    assert L.yy_set_allocator(None, half, FREE_FN(), None) == -2                 # YY_EINVAL
    assert L.yy_set_allocator(None, ALLOC_FN(), FREE_FN(), None) == 0
