"""Device-resident entry points over torch CUDA tensors.

PyTorch is plumbing here: it owns HBM allocations and streams; every byte of
compute runs in ``libebisu.so`` (``ebisu_run_device``,
``ebisu_random_grid_device``, ``ebisu_compare_device``).
"""

from __future__ import annotations

import ctypes

from . import _native
from .shapes import StencilShape


def _torch():
    import torch

    return torch


def _stream_ptr(stream=None) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _check_tensor(x, name, dtype=None):
    torch = _torch()
    dtype = dtype or torch.float64
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == dtype
            and x.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous {str(dtype).split('.')[-1]} CUDA tensor")


def empty_grid(extents, device="cuda"):
    torch = _torch()
    return torch.empty(tuple(int(n) for n in extents), dtype=torch.float64, device=device)


def random_grid_device(extents, seed: int, device="cuda", stream=None):
    """SplitMix64 grid generated in HBM; bit-identical to ``random_grid``."""
    lib = _native.load()
    out = empty_grid(extents, device)
    rc = lib.ebisu_random_grid_device(int(seed) & ((1 << 64) - 1), 0, out.numel(),
                                      out.data_ptr(), _stream_ptr(stream))
    if rc:
        raise _native.NativeError(_native.last_error())
    return out


def sweep_device(d_in, stencil: StencilShape, steps: int, *, out=None, scratch=None, t: int = 0,
                 scheme: int = _native.SCHEME_AUTO, exact: bool = True,
                 persistent: bool = True, stream=None, trace: bool = False, params=None):
    """``steps`` Jacobi steps of the device grid ``d_in`` into ``out``.

    float64 tensors run the reference arithmetic (bitwise in exact mode);
    float32 tensors run the fp32 kernels (north-star tolerance 1e-5).

    Asynchronous on ``stream`` unless ``trace=True`` (then the call waits and
    returns the native counters with the device-measured ``elapsed_ms``).
    """
    torch = _torch()
    if isinstance(d_in, torch.Tensor) and d_in.dtype == torch.float32:
        dtype, run = torch.float32, "ebisu_run_device_f32"  # north-star 1e-5 mode
    else:
        dtype, run = torch.float64, "ebisu_run_device"
    _check_tensor(d_in, "d_in", dtype)
    if steps < 0:
        raise ValueError("step count must be >= 0")
    if d_in.dim() != stencil.dims:
        raise ValueError(f"grid is {d_in.dim()}-D but stencil {stencil.name} is {stencil.dims}-D")
    lib = _native.load()
    if out is None:
        out = _torch().empty_like(d_in)
    _check_tensor(out, "out", dtype)
    if scratch is not None:
        _check_tensor(scratch, "scratch", dtype)
    st = _native.StencilArgs(stencil)
    ext = _native.extents_c(tuple(d_in.shape))
    prm = params if params is not None else _native.make_params(
        scheme=scheme, t=t, exact=exact, persistent=persistent)
    tr = _native.TraceC() if trace else None
    rc = getattr(lib, run)(ctypes.byref(st.c), d_in.dim(), ext, d_in.data_ptr(),
                              out.data_ptr(), scratch.data_ptr() if scratch is not None else None,
                              int(steps), ctypes.byref(prm), _stream_ptr(stream),
                              ctypes.byref(tr) if tr is not None else None)
    if rc:
        msg = _native.last_error()
        if rc == _native.EBISU_ERR_VALUE:
            raise ValueError(msg)
        raise _native.NativeError(f"libebisu error {rc}: {msg}")
    if trace:
        d = tr.to_dict()
        d["kernel"] = _native.kernel_name(tr.kernel_id)
        d["arith"] = _native.ARITH_NAMES.get(tr.arith, str(tr.arith))
        return out, d
    return out


def compare_device(a, b, stream=None) -> dict:
    """Bitwise + max-abs comparison of two device arrays, on the device."""
    _check_tensor(a, "a")
    _check_tensor(b, "b")
    if a.shape != b.shape:
        raise ValueError("shape mismatch")
    lib = _native.load()
    m = ctypes.c_int64()
    f = ctypes.c_int64()
    mx = ctypes.c_double()
    mr = ctypes.c_double()
    rc = lib.ebisu_compare_device(a.data_ptr(), b.data_ptr(), a.numel(), ctypes.byref(m),
                                  ctypes.byref(f), ctypes.byref(mx), ctypes.byref(mr),
                                  _stream_ptr(stream))
    if rc:
        raise _native.NativeError(_native.last_error())
    return {"mismatches": m.value, "first_mismatch": f.value, "max_abs_diff": mx.value,
            "max_abs_ref": mr.value}
