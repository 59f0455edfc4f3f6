"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of ``liboracle.so``, the plain-C
restatement of the reference sweep (``stencil_oracle.c``; builds with
``make -C oracle``).

Same contract as ``stencil_oracle.reference_run`` (reference grid.py:106-113,
every multiply and add separately rounded, taps in order), multi-threaded
over rows; bitwise equal to the numpy restatement and pinned against the
reference's golden digests by ``tests/test_oracle.py``.  Used to generate
the full-size golden digests (``tests/golden/make_fullsize_golden.py``), as a
parity checker in tests, and by ``bench.py``'s CPU legs.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-C", _HERE, "-s"], check=True)
    return LIB_PATH


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        lib = ctypes.CDLL(LIB_PATH)
        i32, i64, vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
        lib.oracle_run.restype = i32
        lib.oracle_run.argtypes = [i32, vp, i32, vp, vp, vp, vp, i64, i32]
        lib.oracle_uniform.restype = None
        lib.oracle_uniform.argtypes = [ctypes.c_uint64, i64, i64, vp]
        lib.oracle_threads.restype = i32
        _lib = lib
    return _lib


def threads() -> int:
    return int(load().oracle_threads())


def uniform_array(seed: int, n: int, start: int = 0) -> np.ndarray:
    """Draws [start, start+n) of SplitMix64(seed) (reference rng.py:31-46)."""
    out = np.empty(int(n), dtype=np.float64)
    load().oracle_uniform(ctypes.c_uint64(seed & ((1 << 64) - 1)), int(start), int(n),
                          out.ctypes.data)
    return out


def reference_run(cells: np.ndarray, taps, t: int, threads: int = 0) -> np.ndarray:
    """``t``-fold composition of reference_step over ``cells`` (float64)."""
    src = np.ascontiguousarray(cells, dtype=np.float64)
    dims = src.ndim
    offs = np.ascontiguousarray(np.array([o for o, _ in taps], dtype=np.int32).reshape(-1))
    coef = np.ascontiguousarray(np.array([c for _, c in taps], dtype=np.float64))
    if offs.size != len(taps) * dims:
        raise ValueError(f"grid is {dims}-D but the taps are not")
    ext = np.array(src.shape, dtype=np.int64)
    out = np.empty_like(src)
    rc = load().oracle_run(dims, ext.ctypes.data, len(taps), offs.ctypes.data, coef.ctypes.data,
                           src.ctypes.data, out.ctypes.data, int(t), int(threads))
    if rc != 0:
        raise ValueError("oracle_run rejected the arguments (extent too small or bad taps)")
    return out
