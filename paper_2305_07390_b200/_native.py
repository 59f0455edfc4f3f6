"""ctypes binding of ``libebisu.so`` (the C ABI in ``include/ebisu.h``).

The shared library is built in-tree (``make -C paper_2305_07390_b200/csrc``
or ``__graft_entry__.build()``).  There is no CPU fallback: if the library is
missing, every compute call raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# EBISU_LIB_PATH lets experiments A/B alternative builds of the same ABI.
LIB_PATH = os.environ.get("EBISU_LIB_PATH") or os.path.join(_HERE, "libebisu.so")

EBISU_OK = 0
EBISU_ERR_VALUE = 1
EBISU_ERR_PARAM = 2
EBISU_ERR_CUDA = 3
EBISU_ERR_UNSUPPORTED = 4
EBISU_ERR_NO_DEVICE = 5

SCHEME_AUTO = 0
SCHEME_NAIVE = 1
SCHEME_SM_TILING = 2
SCHEME_DEVICE_TILING = 3
SCHEME_RESIDENT = 4  # resident tiles, runtime taps (any stencil)

# Every symbol include/ebisu.h declares (checked by tests/test_native_abi.py).
ABI_VERSION = 3  # include/ebisu.h EBISU_ABI_VERSION (ParamsC layout below)

EXPORTS = (
    "ebisu_abi_version",
    "ebisu_last_error",
    "ebisu_kernel_name",
    "ebisu_device_count",
    "ebisu_check_compatible",
    "ebisu_run_host",
    "ebisu_run_device",
    "ebisu_run_host_f32",
    "ebisu_run_device_f32",
    "ebisu_random_grid_device",
    "ebisu_compare_device",
    "ebisu_release_scratch",
)


class NativeUnavailable(RuntimeError):
    """libebisu.so is not built or cannot be loaded."""


class NativeError(RuntimeError):
    """CUDA / unsupported-request failure reported by the library."""


class StencilC(ctypes.Structure):
    _fields_ = [
        ("dims", ctypes.c_int32),
        ("ntaps", ctypes.c_int32),
        ("offsets", ctypes.POINTER(ctypes.c_int32)),
        ("coeffs", ctypes.POINTER(ctypes.c_double)),
    ]


class ParamsC(ctypes.Structure):
    _fields_ = [
        ("scheme", ctypes.c_int32),
        ("t", ctypes.c_int32),
        ("tile", ctypes.c_int32 * 2),
        ("device_tile_grid", ctypes.c_int32 * 2),
        ("lazy", ctypes.c_int32),
        ("exact", ctypes.c_int32),
        ("persistent", ctypes.c_int32),
        ("validate_tile", ctypes.c_int32),
        ("lane_cells", ctypes.c_int32),
        ("seg_rows", ctypes.c_int32),
        ("variant", ctypes.c_int32),
        ("per_tap_products", ctypes.c_int32),
        ("out_planes", ctypes.c_int32 * 2),
        ("frame_ready", ctypes.c_int32),
        ("reserve_sms", ctypes.c_int32),
    ]


class TraceC(ctypes.Structure):
    _fields_ = [
        ("gm_loads", ctypes.c_uint64),
        ("gm_stores", ctypes.c_uint64),
        ("gm_halo_loads", ctypes.c_uint64),
        ("gm_halo_stores", ctypes.c_uint64),
        ("syncs_block", ctypes.c_uint64),
        ("syncs_device", ctypes.c_uint64),
        ("cells_computed", ctypes.c_uint64),
        ("cells_valid", ctypes.c_uint64),
        ("device_tiles", ctypes.c_uint64),
        ("kernel_launches", ctypes.c_uint64),
        ("elapsed_ms", ctypes.c_double),
        ("kernel_id", ctypes.c_int32),
        ("t_used", ctypes.c_int32),
        ("grid_ctas", ctypes.c_int32),
        ("warps_per_cta", ctypes.c_int32),
        ("arith", ctypes.c_int32),
        ("cluster_ctas", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 2),
    ]

    def to_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_ if name != "reserved"}


_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    """Load (once) and type the library; raise NativeUnavailable if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is not built; run `make -C paper_2305_07390_b200/csrc -j8` "
                "(there is no CPU fallback)"
            )
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as e:  # pragma: no cover - depends on the box
            raise NativeUnavailable(f"cannot load {LIB_PATH}: {e}") from e
        i32, i64, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        vp, dp = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)
        lib.ebisu_abi_version.restype = i32
        lib.ebisu_last_error.restype = ctypes.c_char_p
        lib.ebisu_kernel_name.restype = ctypes.c_char_p
        lib.ebisu_kernel_name.argtypes = [i32]
        lib.ebisu_device_count.restype = i32
        lib.ebisu_check_compatible.restype = i32
        lib.ebisu_check_compatible.argtypes = [ctypes.POINTER(StencilC), i32,
                                               ctypes.POINTER(i64), ctypes.POINTER(ParamsC)]
        lib.ebisu_run_host.restype = i32
        lib.ebisu_run_host.argtypes = [ctypes.POINTER(StencilC), i32, ctypes.POINTER(i64),
                                       vp, vp, i64, ctypes.POINTER(ParamsC),
                                       ctypes.POINTER(TraceC)]
        lib.ebisu_run_device.restype = i32
        lib.ebisu_run_device.argtypes = [ctypes.POINTER(StencilC), i32, ctypes.POINTER(i64),
                                         vp, vp, vp, i64, ctypes.POINTER(ParamsC), vp,
                                         ctypes.POINTER(TraceC)]
        lib.ebisu_run_host_f32.restype = i32
        lib.ebisu_run_host_f32.argtypes = lib.ebisu_run_host.argtypes
        lib.ebisu_run_device_f32.restype = i32
        lib.ebisu_run_device_f32.argtypes = lib.ebisu_run_device.argtypes
        lib.ebisu_random_grid_device.restype = i32
        lib.ebisu_random_grid_device.argtypes = [u64, i64, i64, vp, vp]
        lib.ebisu_compare_device.restype = i32
        lib.ebisu_compare_device.argtypes = [vp, vp, i64, ctypes.POINTER(i64),
                                             ctypes.POINTER(i64), dp, dp, vp]
        lib.ebisu_release_scratch.restype = i32
        if lib.ebisu_abi_version() != ABI_VERSION:
            raise NativeUnavailable("libebisu ABI version mismatch")
        _lib = lib
        return lib


def available() -> bool:
    try:
        load()
        return True
    except NativeUnavailable:
        return False


def last_error() -> str:
    return load().ebisu_last_error().decode(errors="replace")


# ebisu_trace.arith (include/ebisu.h EBISU_ARITH_*)
ARITH_NAMES = {0: "shared_products", 1: "per_tap_exact", 2: "per_tap_fma", 3: "reassociated"}


def kernel_name(kid: int) -> str:
    return load().ebisu_kernel_name(kid).decode()


def device_count() -> int:
    return int(load().ebisu_device_count())


class StencilArgs:
    """Keeps the ctypes views (and their backing arrays) alive for one call."""

    def __init__(self, stencil):
        offs = np.ascontiguousarray(np.array(stencil.offsets, dtype=np.int32).reshape(-1))
        coef = np.ascontiguousarray(np.array(stencil.coefficients, dtype=np.float64))
        self._offs, self._coef = offs, coef
        self.c = StencilC(
            stencil.dims,
            len(stencil.taps),
            offs.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            coef.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
        )


def make_params(scheme: int = SCHEME_AUTO, t: int = 0, tile=(0, 0), device_tile_grid=(0, 0),
                lazy: bool = False, exact: bool = True, persistent: bool = True,
                validate_tile: bool = False, lane_cells: int = 0,
                seg_rows: int = 0, variant: int = 0,
                per_tap_products: bool = False, out_planes=(0, 0),
                frame_ready: bool = False, reserve_sms: int = 0) -> ParamsC:
    p = ParamsC()
    p.scheme = scheme
    p.t = int(t)
    tile = tuple(tile) + (0, 0)
    p.tile[0], p.tile[1] = int(tile[0]), int(tile[1])
    g = tuple(device_tile_grid or ()) + (0, 0)
    p.device_tile_grid[0], p.device_tile_grid[1] = int(g[0]), int(g[1])
    p.lazy = int(bool(lazy))
    p.exact = int(bool(exact))
    p.persistent = int(bool(persistent))
    p.validate_tile = int(bool(validate_tile))
    p.lane_cells = int(lane_cells)
    p.seg_rows = int(seg_rows)
    p.variant = int(variant)
    p.per_tap_products = int(bool(per_tap_products))
    p.out_planes[0], p.out_planes[1] = int(out_planes[0]), int(out_planes[1])
    p.frame_ready = int(bool(frame_ready))
    p.reserve_sms = int(reserve_sms)
    return p


def extents_c(extents):
    arr = (ctypes.c_int64 * len(extents))(*[int(n) for n in extents])
    return arr
