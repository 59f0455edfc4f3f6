"""B200 engine for stencilplan: a self-contained ctypes binding of libebisu.so.

This file is the reference-side binding INTEGRATION.md §2 documents (it is
included there verbatim and a GPU test imports and runs this very file):
a stencilplan maintainer drops it in as ``stencilplan/engine/b200.py`` and
adds one registry line (planner.py:219).  It depends only on numpy, ctypes
and stencilplan -- not on the paper_2305_07390_b200 Python package.

``run_b200(grid, stencil, params, steps=None)`` keeps the engine contract of
``run_sm_tiling`` (engine/sm.py:51): returns ``(Grid, ExecutionTrace)``, the
result bitwise equal to ``reference_run(grid, stencil, steps)``
(grid.py:106-113); bad parameters raise ``ParamError``, bad grids
``ValueError``, with the reference's messages.  The trace holds the GPU
kernel geometry's own counters (for the reference's tile-semantics
counters use ``paper_2305_07390_b200.stencilplan_bridge``).
"""

import ctypes
import os

import numpy as np
from stencilplan.engine.params import ParamError
from stencilplan.engine.trace import ExecutionTrace
from stencilplan.grid import Grid, _check_compatible

_LIB = os.environ.get("EBISU_LIB", "libebisu.so")


class _Stencil(ctypes.Structure):  # ebisu_stencil (include/ebisu.h)
    _fields_ = [("dims", ctypes.c_int32), ("ntaps", ctypes.c_int32),
                ("offsets", ctypes.POINTER(ctypes.c_int32)),
                ("coeffs", ctypes.POINTER(ctypes.c_double))]


class _Params(ctypes.Structure):  # ebisu_params
    _fields_ = [("scheme", ctypes.c_int32), ("t", ctypes.c_int32),
                ("tile", ctypes.c_int32 * 2), ("device_tile_grid", ctypes.c_int32 * 2),
                ("lazy", ctypes.c_int32), ("exact", ctypes.c_int32),
                ("persistent", ctypes.c_int32), ("validate_tile", ctypes.c_int32),
                ("lane_cells", ctypes.c_int32), ("seg_rows", ctypes.c_int32),
                ("variant", ctypes.c_int32), ("per_tap_products", ctypes.c_int32),
                ("out_planes", ctypes.c_int32 * 2), ("frame_ready", ctypes.c_int32),
                ("reserve_sms", ctypes.c_int32)]


class _Trace(ctypes.Structure):  # ebisu_trace
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "gm_loads", "gm_stores", "gm_halo_loads", "gm_halo_stores", "syncs_block",
        "syncs_device", "cells_computed", "cells_valid", "device_tiles",
        "kernel_launches")] + [("elapsed_ms", ctypes.c_double)] + [
        (n, ctypes.c_int32) for n in ("kernel_id", "t_used", "grid_ctas",
                                      "warps_per_cta", "arith", "cluster_ctas")] + [
        ("reserved", ctypes.c_int32 * 2)]


_lib = ctypes.CDLL(_LIB)
_lib.ebisu_last_error.restype = ctypes.c_char_p
_lib.ebisu_run_host.restype = ctypes.c_int32
# full prototypes: without argtypes ctypes would pass the 64-bit buffer
# addresses and the int64 step count as 32-bit C ints
_lib.ebisu_run_host.argtypes = [
    ctypes.POINTER(_Stencil), ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(_Params),
    ctypes.POINTER(_Trace)]

_SCHEMES = {"sm-tiling": 2, "device-tiling": 3}


def run_b200(grid, stencil, params, steps=None):
    _check_compatible(grid, stencil)
    if params.scheme not in _SCHEMES:
        raise ParamError(f"unknown scheme {params.scheme!r}")
    steps = params.t if steps is None else int(steps)
    offs = np.ascontiguousarray(np.array(stencil.offsets, dtype=np.int32).ravel())
    coef = np.ascontiguousarray(np.array(stencil.coefficients, dtype=np.float64))
    st = _Stencil(stencil.dims, len(stencil.taps),
                  offs.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                  coef.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    prm = _Params(scheme=_SCHEMES[params.scheme], t=params.t, exact=1, persistent=1,
                  validate_tile=1)
    for i, w in enumerate(tuple(params.tile)[:2]):
        prm.tile[i] = int(w)
    for i, g in enumerate(tuple(params.device_tile_grid or ())[:2]):
        prm.device_tile_grid[i] = int(g)
    src = np.ascontiguousarray(grid.cells, dtype=np.float64)
    out = np.empty_like(src)
    ext = (ctypes.c_int64 * src.ndim)(*src.shape)
    tr = _Trace()
    rc = _lib.ebisu_run_host(ctypes.byref(st), src.ndim, ext, src.ctypes.data,
                             out.ctypes.data, steps, ctypes.byref(prm), ctypes.byref(tr))
    if rc == 1:
        raise ValueError(_lib.ebisu_last_error().decode())
    if rc == 2:
        raise ParamError(_lib.ebisu_last_error().decode())
    if rc:
        raise RuntimeError(_lib.ebisu_last_error().decode())
    trace = ExecutionTrace(gm_loads=tr.gm_loads, gm_stores=tr.gm_stores,
                           syncs_block=tr.syncs_block, syncs_device=tr.syncs_device,
                           cells_computed=tr.cells_computed, cells_valid=tr.cells_valid,
                           device_tiles=tr.device_tiles)
    return Grid(out, grid.boundary), trace
