"""CPU checks of the boundary: libcabs.so loads and exports every symbol that
include/cabs.h declares, with the binding's signatures (no compute calls)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "cabs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cabs_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_six_entry_points():
    names = _declared()
    for f in ("cabs_pilot", "cabs_embed", "cabs_kmeans", "cabs_select", "cabs_sketch", "cabs_residual"):
        assert f in names


def test_library_exports_every_declared_symbol():
    from paper_1607_07395_b200 import build, cabs
    build.build()
    L = ctypes.CDLL(build.LIB)
    for name in _declared():
        assert hasattr(L, name), name
    assert set(_declared()) == set(cabs.exported_symbols())
    cabs.load()


def test_sm100a_code_only():
    from paper_1607_07395_b200 import build
    import shutil
    import subprocess
    cuobj = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([cuobj, "--list-elf", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_side_argument_checks_without_gpu():
    """Synchronous argument checks run before any CUDA call, so they work on a CPU box."""
    from paper_1607_07395_b200 import cabs as C
    L = C.load()
    p = C.Plan(100, 80, 0, 100, 0, 80, 10, 0, 1)
    assert L.cabs_workspace_bytes(ctypes.byref(p)) > 0
    bad = C.Plan(100, 80, 0, 100, 0, 80, 2000, 0, 1)  # kmax > CABS_KMAX
    assert L.cabs_workspace_bytes(ctypes.byref(bad)) == 0
    assert C.cabs_padded_ld(50) == 64 and C.cabs_padded_ld(1) == 32
    st = L.cabs_pilot(ctypes.byref(p), None, 5, 0, None, None, None, 0, None, 0, None, 0, None, 0, None, None)
    assert st == 6  # CABS_ERR_WORKSPACE (ws NULL) -- checked before the source
    assert C.cabs_version() == (0, 1)
    assert L.cabs_status_string(1) == b"invalid argument"
