"""The C-ABI library loads and exports every symbol include/ebisu.h declares;
validation entry points work without a GPU (no compute calls here)."""

from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2305_07390_b200 import _native
from paper_2305_07390_b200.shapes import make_benchmark

HEADER = os.path.join(ROOT, "include", "ebisu.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"EBISU_API\s+[\w\s\*]+?\b(ebisu_\w+)\s*\(", text)))


def test_header_lists_match_binding():
    assert declared_symbols() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libebisu.so not built")
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (ebisu_\w+)", out))
    missing = set(declared_symbols()) - exported
    assert not missing, missing
    # nothing beyond the ABI leaks (static cudart is hidden)
    assert exported == set(declared_symbols())
    lib = _native.load()
    for name in declared_symbols():
        assert hasattr(lib, name)


def test_abi_version_and_kernel_names():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libebisu.so not built")
    lib = _native.load()
    assert lib.ebisu_abi_version() == 3
    assert _native.kernel_name(2) == "stream2d_tb"
    assert _native.kernel_name(1) == "naive_step"


def _check(name, extents, **kw):
    lib = _native.load()
    st = _native.StencilArgs(make_benchmark(name))
    ext = _native.extents_c(extents)
    prm = _native.make_params(**kw)
    return lib.ebisu_check_compatible(ctypes.byref(st.c), len(extents), ext, ctypes.byref(prm))


def test_native_validation_messages():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libebisu.so not built")
    assert _check("j2d5pt", (10, 10)) == _native.EBISU_OK
    assert _check("j2d5pt", (10,)) == _native.EBISU_ERR_VALUE
    assert "2-D" in _native.last_error()
    assert _check("j2d9pt", (4, 10)) == _native.EBISU_ERR_VALUE
    assert "too small" in _native.last_error()
    rc = _check("j2d5pt", (12, 20), scheme=_native.SCHEME_SM_TILING, t=5, tile=(10, 0),
                validate_tile=True)
    assert rc == _native.EBISU_ERR_PARAM and "valid core" in _native.last_error()


def test_run_without_device_fails_loudly():
    if not os.path.exists(_native.LIB_PATH):
        pytest.skip("libebisu.so not built")
    if _native.device_count() > 0:
        pytest.skip("GPU visible")
    import numpy as np

    lib = _native.load()
    st = _native.StencilArgs(make_benchmark("j2d5pt"))
    a = np.zeros((8, 8))
    b = np.zeros((8, 8))
    prm = _native.make_params()
    rc = lib.ebisu_run_host(ctypes.byref(st.c), 2, _native.extents_c((8, 8)), a.ctypes.data,
                            b.ctypes.data, 3, ctypes.byref(prm), None)
    assert rc == _native.EBISU_ERR_NO_DEVICE


def test_integration_binding_is_the_tested_file():
    """INTEGRATION.md §2 shows tools/stencilplan_b200_engine.py verbatim (the
    file the GPU suite runs against the reference), with argtypes declared."""
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    a = doc.index("<!-- BEGIN tools/stencilplan_b200_engine.py -->")
    b = doc.index("<!-- END tools/stencilplan_b200_engine.py -->")
    block = doc[a:b].split("```python\n", 1)[1].rsplit("```", 1)[0]
    src = open(os.path.join(ROOT, "tools", "stencilplan_b200_engine.py")).read()
    assert block == src
    assert "_lib.ebisu_run_host.argtypes" in src
