"""Tiling engines on the B200 (drop-in for ``stencilplan.engine``).

Same registry shape as the reference (``planner._ENGINES``, planner.py:219):
``engine(grid, stencil, params) -> (Grid, ExecutionTrace)``, output equal to
``reference_run(grid, stencil, params.t)`` (planner.py:227-232), ``ParamError``
for invalid parameters with the reference's messages (engine/params.py:52-90,
engine/sm.py:39-48, engine/device.py:43-52).

The reference engines *simulate* the two EBISU schemes on the CPU with access
accounting.  Here the scheme runs as real sm_100a kernels.  The returned
``ExecutionTrace`` carries the counters the reference engine would emit for
the caller's ``TilingParams`` (``accounting.py``: exact closed forms of
engine/sm.py and engine/device.py under the trace.py:1-17 conventions, so
``trace_summary``, the planner and the reference's accounting tests read it
unchanged), and in ``trace.gpu`` the facts of the run that actually
happened: kernel family, fused depth, launches, device time and the GPU
geometry's own counters (cells loaded/stored by TMA, lanes computed, work
units, grid-wide barriers).
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from fractions import Fraction

from . import _native, accounting
from .grid import Grid, sweep
from .shapes import StencilShape

SM_TILING = "sm-tiling"
DEVICE_TILING = "device-tiling"
SCHEMES = (SM_TILING, DEVICE_TILING)
ITEMS_PER_THREAD = 4


class ParamError(ValueError):
    """Invalid tiling parameters (engine/params.py:15)."""


@dataclass
class TilingParams:
    """Reference ``TilingParams`` (engine/params.py:18-90)."""

    scheme: str
    t: int
    tile: tuple[int, ...]
    device_tile_grid: tuple[int, ...] | None = None
    lazy: bool = False
    rst: bool = False
    prefetch: bool = False
    transpose_halo: bool = False
    queue_variant: str | None = None
    workers: int = 1

    def __post_init__(self):
        if self.scheme not in SCHEMES:
            raise ParamError(f"unknown scheme {self.scheme!r}")
        if self.t < 1:
            raise ParamError("temporal depth must be >= 1")
        self.tile = tuple(int(x) for x in self.tile)
        if self.device_tile_grid is not None:
            self.device_tile_grid = tuple(int(x) for x in self.device_tile_grid)

    def tiled_axes(self, dims: int) -> tuple[int, ...]:
        if dims == 1:
            return (0,)
        if dims == 2 and self.scheme == DEVICE_TILING:
            return (0, 1)
        return tuple(range(1, dims))

    def validate(self, stencil: StencilShape, extents: tuple[int, ...]):
        dims, rad, t = stencil.dims, stencil.radius, self.t
        axes = self.tiled_axes(dims)
        if len(self.tile) != len(axes):
            raise ParamError(
                f"{dims}-D {self.scheme} needs {len(axes)} tile extents, got {len(self.tile)}"
            )
        if self.scheme == SM_TILING:
            for w in self.tile:
                if w - 2 * rad * t <= 0:
                    raise ParamError(
                        f"tile extent {w} leaves no valid core at depth {t} "
                        f"(needs > {2 * rad * t})"
                    )
            return
        grid = self.device_tile_grid or (1,) * len(axes)
        if len(grid) != len(axes):
            raise ParamError(f"device tile grid needs {len(axes)} entries, got {len(grid)}")
        halo = rad * t
        for g, w, axis in zip(grid, self.tile, axes):
            if g < 1:
                raise ParamError("device tile grid entries must be >= 1")
            interior = extents[axis] - 2 * rad
            loaded = g * w
            if loaded < interior and loaded + 2 * halo > extents[axis]:
                raise ParamError(
                    f"device tile of {loaded} cells plus 2*{halo} halo "
                    f"exceeds extent {extents[axis]} on axis {axis}"
                )
            if loaded - 2 * halo <= 0 and loaded < interior:
                raise ParamError(f"device tile of {loaded} cells has no core at depth {t}")


# ---------------------------------------------------------------------------
# on-chip access model (engine/rst.py:23-51) -- measurement only
# ---------------------------------------------------------------------------

def rst_shared_per_cell(stencil: StencilShape, ipt: int = ITEMS_PER_THREAD) -> Fraction:
    """engine/rst.py:26-45."""
    return accounting.rst_shared_per_cell(stencil.offsets, stencil.dims, ipt)


def onchip_charges(stencil: StencilShape, rst: bool) -> tuple[Fraction, Fraction]:
    """engine/rst.py:48-51."""
    return accounting.onchip_charges(stencil.offsets, stencil.dims, rst)


# ---------------------------------------------------------------------------
# traces (engine/trace.py)
# ---------------------------------------------------------------------------

@dataclass
class ExecutionTrace:
    gm_loads: int = 0
    gm_stores: int = 0
    gm_halo_loads: int = 0
    gm_halo_stores: int = 0
    onchip_shared: Fraction = Fraction(0)
    onchip_register: Fraction = Fraction(0)
    syncs_block: int = 0
    syncs_device: int = 0
    cells_computed: int = 0
    cells_valid: int = 0
    device_tiles: int = 0
    halo_transactions: int = 0
    wall_phases: list = field(default_factory=list)
    # GPU facts (not in the reference trace): what ran and the kernel
    # geometry's own counters (native ebisu_trace)
    kernel: str = ""
    t_used: int = 0
    elapsed_ms: float = 0.0
    kernel_launches: int = 0
    gpu: dict = field(default_factory=dict)

    PHASE_CAP = accounting.PHASE_CAP

    def charge_compute(self, lanes: int, shared_pc: Fraction, register_pc: Fraction):
        self.cells_computed += lanes
        self.onchip_shared += shared_pc * lanes
        self.onchip_register += register_pc * lanes

    def phase(self, tag: str, cells: int):
        if len(self.wall_phases) < self.PHASE_CAP:
            self.wall_phases.append((tag, cells))
        elif len(self.wall_phases) == self.PHASE_CAP:
            self.wall_phases.append(("truncated", 1))

    def merge(self, other: "ExecutionTrace"):
        for f in ("gm_loads", "gm_stores", "gm_halo_loads", "gm_halo_stores", "onchip_shared",
                  "onchip_register", "syncs_block", "syncs_device", "cells_computed",
                  "cells_valid", "device_tiles", "halo_transactions", "kernel_launches"):
            setattr(self, f, getattr(self, f) + getattr(other, f))

    def to_dict(self) -> dict:
        return {
            "gm_loads": self.gm_loads,
            "gm_stores": self.gm_stores,
            "gm_halo_loads": self.gm_halo_loads,
            "gm_halo_stores": self.gm_halo_stores,
            "onchip_accesses": {
                "shared-level": float(self.onchip_shared),
                "register-level": float(self.onchip_register),
            },
            "syncs": {"block": self.syncs_block, "device": self.syncs_device},
            "cells_computed": self.cells_computed,
            "cells_valid": self.cells_valid,
            "device_tiles": self.device_tiles,
            "halo_transactions": self.halo_transactions,
            "wall_phases": [[tag, n] for tag, n in self.wall_phases],
            "gpu": dict(self.gpu, kernel=self.kernel, t_used=self.t_used,
                        elapsed_ms=self.elapsed_ms, kernel_launches=self.kernel_launches),
        }

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True, indent=2) + "\n"

    def phases_csv(self) -> str:
        lines = ["phase,cells"] + [f"{tag},{n}" for tag, n in self.wall_phases]
        return "\n".join(lines) + "\n"


@dataclass
class AccountingReport:
    a_gm_measured: float
    a_sm_measured: float
    valid_proportion_measured: float
    valid_proportion_model: float | None
    syncs_block: int
    syncs_device: int
    device_tiles: int

    def to_dict(self) -> dict:
        return {
            "a_gm_measured": self.a_gm_measured,
            "a_sm_measured": self.a_sm_measured,
            "valid_proportion_measured": self.valid_proportion_measured,
            "valid_proportion_model": self.valid_proportion_model,
            "syncs": {"block": self.syncs_block, "device": self.syncs_device},
            "device_tiles": self.device_tiles,
        }


def trace_summary(trace: ExecutionTrace, stencil: StencilShape, params: TilingParams, domain,
                  two_sided: bool = True) -> AccountingReport:
    """Reference ``trace_summary`` (engine/summary.py:10-38)."""
    if trace.cells_computed == 0 or trace.cells_valid == 0:
        raise ValueError("empty trace: no computed or valid cells")
    a_gm = (trace.gm_loads + trace.gm_stores) / trace.cells_valid
    a_sm = float(trace.onchip_shared / trace.cells_computed)
    v_meas = trace.cells_valid / trace.cells_computed
    v_model = None
    if params.scheme == SM_TILING:
        k = 2 if two_sided else 1
        v_model = 1.0
        for w in params.tile:
            v_model *= (w - k * params.t * stencil.radius) / w
    return AccountingReport(a_gm, a_sm, v_meas, v_model, trace.syncs_block, trace.syncs_device,
                            trace.device_tiles)


# ---------------------------------------------------------------------------
# engines
# ---------------------------------------------------------------------------

def _check(grid: Grid, stencil: StencilShape, params: TilingParams, scheme: str, fname: str):
    if params.scheme != scheme:
        raise ParamError(f"{fname} got scheme {params.scheme!r}")
    if grid.dims != stencil.dims:
        raise ParamError("grid/stencil dimensionality mismatch")
    rad = stencil.radius
    for n in grid.extents:
        if n <= 2 * rad:
            raise ParamError(f"extent {n} too small for radius {rad}")
    params.validate(stencil, grid.extents)


def _reference_trace(stencil: StencilShape, extents, params: TilingParams,
                     steps: int) -> ExecutionTrace:
    """Counters the reference engine emits for ``params`` (one epoch of
    ``params.t`` steps, accounting.py); ``steps`` beyond one epoch add one
    epoch's counters per further ``params.t`` steps (a shorter last epoch is
    counted at its own depth)."""
    import dataclasses

    trace = ExecutionTrace()
    offs = [tuple(o) for o in stencil.offsets]
    done = 0
    while done < steps:
        depth = min(params.t, steps - done)
        p = params if depth == params.t else dataclasses.replace(params, t=depth)
        c = accounting.reference_counters(offs, stencil.dims, extents, p)
        for f in ("gm_loads", "gm_stores", "gm_halo_loads", "gm_halo_stores", "onchip_shared",
                  "onchip_register", "syncs_block", "syncs_device", "cells_computed",
                  "cells_valid", "device_tiles", "halo_transactions"):
            setattr(trace, f, getattr(trace, f) + getattr(c, f))
        for tag, n in c.wall_phases:
            if tag != "truncated":
                trace.phase(tag, n)
            elif len(trace.wall_phases) == trace.PHASE_CAP:
                trace.phase(tag, n)
        done += depth
    return trace


def _run(grid, stencil, params, scheme_code, steps=None, exact=True):
    steps = params.t if steps is None else steps
    out, tr = sweep(grid, stencil, steps, t=params.t, scheme=scheme_code, exact=exact,
                    trace=True, exc_param=ParamError)
    trace = _reference_trace(stencil, grid.extents, params, steps)
    if tr is not None:
        trace.kernel = tr["kernel"]
        trace.t_used = tr["t_used"]
        trace.elapsed_ms = tr["elapsed_ms"]
        trace.kernel_launches = tr["kernel_launches"]
        trace.gpu = {k: tr[k] for k in ("gm_loads", "gm_stores", "gm_halo_loads",
                                        "gm_halo_stores", "syncs_block", "syncs_device",
                                        "cells_computed", "cells_valid", "device_tiles",
                                        "grid_ctas", "warps_per_cta")}
    return out, trace


def run_sm_tiling(grid: Grid, stencil: StencilShape, params: TilingParams, *, steps=None,
                  exact: bool = True):
    """Overlapped temporal blocking on the B200 (reference engine/sm.py:51)."""
    _check(grid, stencil, params, SM_TILING, "run_sm_tiling")
    return _run(grid, stencil, params, _native.SCHEME_SM_TILING, steps, exact)


def run_device_tiling(grid: Grid, stencil: StencilShape, params: TilingParams, *, steps=None,
                      exact: bool = True):
    """Device-tiling entry (reference engine/device.py:55)."""
    _check(grid, stencil, params, DEVICE_TILING, "run_device_tiling")
    return _run(grid, stencil, params, _native.SCHEME_DEVICE_TILING, steps, exact)


ENGINES = {SM_TILING: run_sm_tiling, DEVICE_TILING: run_device_tiling}
