"""Grids and the drop-in sweep (reference ``pkg/src/stencilplan/grid.py``).

``reference_step`` / ``reference_run`` keep the reference signatures and
contract (pure: the input grid is untouched and a new ``Grid`` is returned;
``ValueError`` with the reference messages on bad input), but the sweep runs
on the B200 through ``libebisu.so``:

    reference_run(grid, stencil, t)      grid.py:106-113
    reference_step(grid, stencil)        grid.py:96-103

``sweep`` is the same call with the GPU knobs exposed (fused depth, exact vs
FMA accumulation, persistent cooperative launch).  Exact mode (default)
is bitwise equal to the reference; FMA mode is within 1e-12 relative.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .rng import uniform_array
from .shapes import StencilShape

BOUNDARY_POLICIES = ("fixed-value", "skip-update")


@dataclass
class Grid:
    """Dense N-D float64 cell array with a boundary tag (grid.py:21-49).

    Under both policies the frame (cells within ``radius`` of a face) keeps
    its value; the tags are kept distinct for parity runs.
    """

    cells: np.ndarray
    boundary: str = "fixed-value"

    def __post_init__(self):
        if self.boundary not in BOUNDARY_POLICIES:
            raise ValueError(f"unknown boundary policy {self.boundary!r}")
        self.cells = np.asarray(self.cells, dtype=np.float64)

    @property
    def extents(self) -> tuple[int, ...]:
        return self.cells.shape

    @property
    def dims(self) -> int:
        return self.cells.ndim

    def copy(self) -> "Grid":
        return Grid(self.cells.copy(), self.boundary)


def constant_grid(extents, value: float, boundary: str = "fixed-value") -> Grid:
    return Grid(np.full(tuple(extents), float(value)), boundary)


def random_grid(extents, seed: int, boundary: str = "fixed-value") -> Grid:
    """SplitMix64 uniforms in [0, 1) (grid.py:56-60); bit-identical draws."""
    extents = tuple(int(n) for n in extents)
    n = int(np.prod(extents)) if extents else 1
    return Grid(uniform_array(seed, n).reshape(extents), boundary)


def check_compatible(grid: Grid, stencil: StencilShape):
    """Reference ``_check_compatible`` (grid.py:63-73), same messages."""
    if grid.dims != stencil.dims:
        raise ValueError(
            f"grid is {grid.dims}-D but stencil {stencil.name} is {stencil.dims}-D"
        )
    rad = stencil.radius
    for n in grid.extents:
        if n <= 2 * rad:
            raise ValueError(f"extent {n} too small for radius {rad} (need > {2 * rad})")


def _raise_native(rc: int, exc_param=None):
    msg = _native.last_error()
    if rc == _native.EBISU_ERR_VALUE:
        raise ValueError(msg)
    if rc == _native.EBISU_ERR_PARAM and exc_param is not None:
        raise exc_param(msg)
    raise _native.NativeError(f"libebisu error {rc}: {msg}")


def sweep(grid: Grid, stencil: StencilShape, steps: int, *, t: int = 0,
          scheme: int = _native.SCHEME_AUTO, exact: bool = True, persistent: bool = True,
          trace: bool = False, params=None, exc_param=None, dtype=np.float64):
    """``steps`` Jacobi steps of ``grid`` on the GPU; returns ``Grid`` (and the
    native trace dict when ``trace=True``).

    ``t`` is the temporal depth fused per HBM round trip (0 = planner
    default).  Host buffers go through ``ebisu_run_host`` (H2D, sweep, D2H).
    ``dtype=np.float32`` runs the fp32 kernels (``ebisu_run_host_f32``; the
    north-star 1e-5 mode); the returned ``Grid`` holds those values as float64,
    the reference Grid's type (grid.py:38).
    """
    if steps < 0:
        raise ValueError("step count must be >= 0")
    check_compatible(grid, stencil)
    if steps == 0:
        out = grid.copy()
        return (out, None) if trace else out
    lib = _native.load()
    f32 = np.dtype(dtype) == np.float32
    if not f32 and np.dtype(dtype) != np.float64:
        raise ValueError("dtype must be float64 or float32")
    src = np.ascontiguousarray(grid.cells, dtype=np.float32 if f32 else np.float64)
    dst = np.empty_like(src)
    st = _native.StencilArgs(stencil)
    ext = _native.extents_c(src.shape)
    prm = params if params is not None else _native.make_params(
        scheme=scheme, t=t, exact=exact, persistent=persistent)
    tr = _native.TraceC()
    run = lib.ebisu_run_host_f32 if f32 else lib.ebisu_run_host
    rc = run(ctypes.byref(st.c), src.ndim, ext, src.ctypes.data, dst.ctypes.data, int(steps),
             ctypes.byref(prm), ctypes.byref(tr))
    if rc != _native.EBISU_OK:
        _raise_native(rc, exc_param)
    out = Grid(dst, grid.boundary)
    if trace:
        d = tr.to_dict()
        d["kernel"] = _native.kernel_name(tr.kernel_id)
        d["arith"] = _native.ARITH_NAMES.get(tr.arith, str(tr.arith))
        return out, d
    return out


def reference_step(grid: Grid, stencil: StencilShape) -> Grid:
    """One Jacobi step on the GPU; drop-in for grid.py:96-103."""
    return sweep(grid, stencil, 1)


def reference_run(grid: Grid, stencil: StencilShape, t: int) -> Grid:
    """``t``-fold composition on the GPU; drop-in for grid.py:106-113."""
    return sweep(grid, stencil, t)
