"""Reference-semantics execution counters for the B200 engines.

The reference engines (``stencilplan.engine.sm`` / ``.device``) *simulate*
the EBISU schemes on the CPU and meter every access into an
``ExecutionTrace`` under the conventions of ``engine/trace.py:1-17``.  The
B200 engines execute the sweep as real kernels whose geometry (128-column
warp strips, 32x64 plane tiles, ...) is chosen for the hardware, not from
``TilingParams.tile``.  So that the engine stays a drop-in for the
reference's accounting contract -- ``planner._simulate_one``
(planner.py:222-251), ``trace_summary`` (engine/summary.py:10-38), the
reference's own ``test_engine_sm`` / ``test_engine_device`` /
acceptance c10-c11 assertions -- this module reproduces the counters the
reference engine would emit for the caller's ``TilingParams``, in closed
form from the same control flow:

* ``sm_trace``      mirrors ``run_sm_tiling`` (engine/sm.py:51-206):
  ``_sm_1d`` (:58-92) and ``_sm_streamed`` / ``_stream_block`` (:95-206),
  then ``_coarse_phases`` (:209-213);
* ``device_trace``  mirrors ``run_device_tiling`` (engine/device.py:55-389):
  ``_device_resident`` with ``_resident_tile_bsp`` (:145-211) or
  ``_resident_tile_lazy`` (:214-261), and ``_device_streamed`` /
  ``_streamed_tile`` (:268-389).

The stream-axis control (circular multi-queue readiness, multiqueue.py:
103-211) does not depend on cell values or on a block's position along the
tiled axes, so it is simulated once per (n0, t, rad, lazy) and the per-block
sizes are summed over blocks.  No cell data is touched: the numbers are
exact integers / rationals, equal to what the reference computes.  The
GPU's own counters travel beside them in ``ExecutionTrace.gpu``.
"""

from __future__ import annotations

import itertools
from fractions import Fraction
from functools import lru_cache
from math import prod

SM_TILING = "sm-tiling"
DEVICE_TILING = "device-tiling"
PHASE_CAP = 4096  # engine/trace.py:55


# ---- engine/common.py helpers (geometry only) ------------------------------

def partition_cores(lo: int, hi: int, width: int) -> list[tuple[int, int]]:
    """common.py:14-24: consecutive cores of ``width`` over [lo, hi)."""
    if hi <= lo:
        raise ValueError("empty interior")
    return [(s, min(s + width, hi)) for s in range(lo, hi, width)]


def even_split(lo: int, hi: int, parts: int) -> list[tuple[int, int]]:
    """common.py:27-38: ``parts`` contiguous chunks, sizes differing by <= 1."""
    n = hi - lo
    parts = min(parts, n)
    base, extra = divmod(n, parts)
    out, start = [], lo
    for i in range(parts):
        w = base + (1 if i < extra else 0)
        out.append((start, start + w))
        start += w
    return out


def coalesced_transactions(cells: int, cell_bytes: int, coalesced: bool) -> int:
    """common.py:115-120 (32-byte transactions)."""
    if coalesced:
        return (cells * cell_bytes + 31) // 32
    return cells


def halo_strip_counts(per_axis_splits, rad: int) -> tuple[int, int, int]:
    """device.py:104-124: (cells, raw transactions, transposed transactions)
    exchanged per step across the internal block boundaries."""
    dims = len(per_axis_splits)
    full = [sum(hi - lo for lo, hi in splits) for splits in per_axis_splits]
    cells = raw_tx = posed_tx = 0
    for axis in range(dims):
        internal = len(per_axis_splits[axis]) - 1
        if internal <= 0:
            continue
        cross = prod(full[a] for a in range(dims) if a != axis)
        strip = 2 * rad * cross * internal
        cells += strip
        contiguous = dims == 1 or axis < dims - 1
        raw_tx += coalesced_transactions(strip, 8, contiguous)
        posed_tx += coalesced_transactions(strip, 8, True)
    return cells, raw_tx, posed_tx


# ---- the stream-axis pipeline (multiqueue.py readiness) --------------------

@lru_cache(maxsize=256)
def stream_schedule(n0: int, t: int, rad: int) -> tuple:
    """Per advance k of ``_stream_block`` / ``_streamed_tile``: the sequence of
    events the loop performs.  Event codes: 'L' plane load (level-0 enqueue,
    frame seed, or upper-frame pass-through), 'C<s>' a counted level-s
    update (s + 1 < t: enqueued to the next level; s + 1 == t: stored).

    Queue readiness (multiqueue.py:157-161): a level is ready when its window
    holds 2*rad+1 entries and it was enqueued since the last shuffle.  The
    queue spacing and lazy capacity do not change readiness.
    """
    window = 2 * rad + 1
    fill = [0] * t
    stale = [False] * t
    counts = [0] * t

    def enqueue(level):
        if fill[level] < window:
            fill[level] += 1
        stale[level] = False

    sched = []
    for k in range(n0 + t * rad):
        ev = []
        if k < n0:
            ev.append("L")
            enqueue(0)
        if rad <= k < t * rad:
            ev.append("L")
            enqueue(k // rad)
        for s in range(t):
            pos = rad + counts[s]
            if pos >= n0:
                continue
            if pos >= n0 - rad:
                ev.append("L")
                counted = False
            elif fill[s] >= window and not stale[s]:
                ev.append(f"C{s}")
                counted = True
            else:
                break
            counts[s] += 1
            if s + 1 < t:
                enqueue(s + 1)
            del counted
        for s in range(t):
            stale[s] = True
        sched.append(tuple(ev))
    return tuple(sched)


def _schedule_totals(n0: int, t: int, rad: int) -> tuple[int, int, int, int]:
    """(plane loads, counted updates, counted updates feeding a next level,
    stores) of one streamed block."""
    loads = comp = fwd = stores = 0
    for ev in stream_schedule(n0, t, rad):
        for e in ev:
            if e == "L":
                loads += 1
            else:
                comp += 1
                if int(e[1:]) + 1 < t:
                    fwd += 1
                else:
                    stores += 1
    return loads, comp, fwd, stores


# ---- on-chip charges (engine/rst.py) ----------------------------------------

def rst_shared_per_cell(offsets, dims: int, ipt: int = 4) -> Fraction:
    """rst.py:26-45."""
    if dims == 1:
        return Fraction(2)
    if dims == 2:
        return Fraction(2) + Fraction(len({o[1] for o in offsets if o[1] != 0}))
    own = {(i, 0) for i in range(ipt)}
    needed = {(o[1] + i, o[2]) for o in offsets for i in range(ipt)}
    return Fraction(2) + Fraction(len(needed - own), ipt)


def onchip_charges(offsets, dims: int, rst: bool) -> tuple[Fraction, Fraction]:
    """rst.py:48-51: (shared-level, register-level) accesses per cell update."""
    total = Fraction(len(offsets) + 1)
    if not rst:
        return total, Fraction(0)
    shared = rst_shared_per_cell(offsets, dims)
    return shared, total - shared


# ---- counters ----------------------------------------------------------------

class Counters:
    """The reference ExecutionTrace fields (trace.py:25-38)."""

    __slots__ = ("gm_loads", "gm_stores", "gm_halo_loads", "gm_halo_stores", "onchip_shared",
                 "onchip_register", "syncs_block", "syncs_device", "cells_computed",
                 "cells_valid", "device_tiles", "halo_transactions", "wall_phases")

    def __init__(self):
        for f in self.__slots__:
            setattr(self, f, 0)
        self.onchip_shared = Fraction(0)
        self.onchip_register = Fraction(0)
        self.wall_phases = []

    def phase(self, tag: str, cells: int):
        if len(self.wall_phases) < PHASE_CAP:
            self.wall_phases.append((tag, cells))
        elif len(self.wall_phases) == PHASE_CAP:
            self.wall_phases.append(("truncated", 1))

    def charge(self, lanes: int, shared_pc: Fraction, reg_pc: Fraction):
        self.cells_computed += lanes
        self.onchip_shared += shared_pc * lanes
        self.onchip_register += reg_pc * lanes


def _coarse_phases(c: Counters, prefetch: bool):
    """sm.py:209-213."""
    c.phase("prefetch-load" if prefetch else "load", c.gm_loads)
    c.phase("compute", c.cells_computed)
    c.phase("store", c.gm_stores)


def sm_trace(offsets, dims: int, extents, params) -> Counters:
    """Counters of ``run_sm_tiling`` (engine/sm.py:51-213) for one epoch of
    ``params.t`` steps."""
    rad = max(abs(v) for o in offsets for v in o)
    t = params.t
    shared_pc, reg_pc = onchip_charges(offsets, dims, params.rst)
    c = Counters()
    if dims == 1:
        # _sm_1d (sm.py:58-92)
        n = extents[0]
        tile = params.tile[0]
        for clo, chi in partition_cores(rad, n - rad, tile - 2 * rad * t):
            lo, hi = max(0, clo - rad * t), min(n, chi + rad * t)
            c.gm_loads += hi - lo
            c.charge(tile * t, shared_pc, reg_pc)
            c.syncs_block += t
            c.gm_stores += chi - clo
            c.cells_valid += (chi - clo) * t
        _coarse_phases(c, params.prefetch)
        return c
    # _sm_streamed / _stream_block (sm.py:95-206)
    n0 = extents[0]
    tiled = extents[1:]
    cores_per_axis = [partition_cores(rad, n - rad, w - 2 * rad * t)
                      for n, w in zip(tiled, params.tile)]
    loads, comp, _fwd, stores = _schedule_totals(n0, t, rad)
    lanes = prod(params.tile)
    advances = n0 + t * rad
    for core_ranges in itertools.product(*cores_per_axis):
        loaded = [(max(0, lo - rad * t), min(n, hi + rad * t))
                  for (lo, hi), n in zip(core_ranges, tiled)]
        loaded_cells = prod(hi - lo for lo, hi in loaded)
        core_cells = prod(hi - lo for lo, hi in core_ranges)
        c.gm_loads += loads * loaded_cells
        c.charge(comp * lanes, shared_pc, reg_pc)
        c.gm_stores += stores * core_cells
        c.cells_valid += stores * core_cells * t
        c.syncs_block += advances * (1 if params.lazy else t)
    _coarse_phases(c, params.prefetch)
    return c


def _tile_cores(extents, tile_spans, rad: int, halo: int):
    """device.py:66-79."""
    cores_per_axis = []
    for n, span in zip(extents, tile_spans):
        interior = n - 2 * rad
        core_w = span if span >= interior else span - 2 * halo
        if core_w <= 0:
            raise ValueError(f"device tile span {span} has no core with halo {halo}")
        cores_per_axis.append(partition_cores(rad, n - rad, core_w))
    return cores_per_axis


def _loaded_range(core, halo, n):
    lo, hi = core
    return max(0, lo - halo), min(n, hi + halo)


def device_trace(offsets, dims: int, extents, params) -> Counters:
    """Counters of ``run_device_tiling`` (engine/device.py:55-389) for one
    epoch of ``params.t`` steps."""
    rad = max(abs(v) for o in offsets for v in o)
    t = params.t
    shared_pc, reg_pc = onchip_charges(offsets, dims, params.rst)
    halo = rad * t
    c = Counters()
    load_tag = "prefetch-load" if params.prefetch else "load"
    if dims <= 2:
        # _device_resident (device.py:85-98)
        grid_shape = params.device_tile_grid or (1,) * dims
        tile_spans = [g * w for g, w in zip(grid_shape, params.tile)]
        cores_per_axis = _tile_cores(extents, tile_spans, rad, halo)
        for tile_core in itertools.product(*cores_per_axis):
            loaded = [_loaded_range(core, halo, n) for core, n in zip(tile_core, extents)]
            if params.lazy:
                _resident_lazy(c, extents, rad, t, loaded, tile_core, grid_shape,
                               shared_pc, reg_pc)
            else:
                _resident_bsp(c, rad, t, loaded, tile_core, grid_shape, shared_pc, reg_pc,
                              load_tag, params.transpose_halo)
            c.device_tiles += 1
        return c
    # _device_streamed / _streamed_tile (device.py:268-389)
    n0 = extents[0]
    tiled = extents[1:]
    grid_shape = params.device_tile_grid or (1, 1)
    tile_spans = [g * w for g, w in zip(grid_shape, params.tile)]
    cores_per_axis = _tile_cores(tiled, tile_spans, rad, halo)
    sched = stream_schedule(n0, t, rad)
    for tile_core in itertools.product(*cores_per_axis):
        loaded = [_loaded_range(co, halo, n) for co, n in zip(tile_core, tiled)]
        per_axis = [even_split(lo, hi, g) for (lo, hi), g in zip(loaded, grid_shape)]
        regions = list(itertools.product(*per_axis))
        halo_cells, raw_tx, posed_tx = halo_strip_counts(per_axis, rad)
        tx = posed_tx if params.transpose_halo else raw_tx
        plane_load = sum(prod(hi - lo + 2 * rad for lo, hi in region) for region in regions)
        lanes = sum(prod(hi - lo for lo, hi in region) for region in regions)
        core_cells = prod(chi - clo for clo, chi in tile_core)
        for ev in sched:
            c.phase(load_tag, plane_load)
            for e in ev:
                if e == "L":
                    c.gm_loads += plane_load
                    continue
                s = int(e[1:])
                c.charge(lanes, shared_pc, reg_pc)
                c.phase("compute", lanes)
                if s + 1 < t:
                    c.gm_stores += halo_cells
                    c.gm_loads += halo_cells
                    c.gm_halo_stores += halo_cells
                    c.gm_halo_loads += halo_cells
                    c.phase("push-halo", halo_cells)
                    c.phase("pull-halo", halo_cells)
                    c.halo_transactions += tx
                else:
                    c.gm_stores += core_cells
                    c.cells_valid += core_cells * t
                    c.phase("store", core_cells)
            if params.lazy:
                c.syncs_device += 1
                c.phase("device-sync", 0)
            else:
                c.syncs_device += t
                for _ in range(t):
                    c.phase("device-sync", 0)
            c.syncs_block += len(regions) * (1 if params.lazy else t)
            c.device_tiles += 1
    return c


def _resident_bsp(c, rad, t, loaded, tile_core, grid_shape, shared_pc, reg_pc, load_tag,
                  transpose_halo):
    """device.py:145-211."""
    per_axis = [even_split(lo, hi, g) for (lo, hi), g in zip(loaded, grid_shape)]
    regions = list(itertools.product(*per_axis))
    size = prod(hi - lo for lo, hi in loaded)
    c.gm_loads += size
    c.phase(load_tag, size)
    halo_cells, raw_tx, posed_tx = halo_strip_counts(per_axis, rad)
    sizes = [prod(hi - lo for lo, hi in region) for region in regions]
    for _ in range(t):
        for s in sizes:
            c.charge(s, shared_pc, reg_pc)
        c.phase("update", int(sum(sizes)))
        c.syncs_block += len(regions)
        c.phase("block-sync", 0)
        c.gm_stores += halo_cells
        c.gm_halo_stores += halo_cells
        c.phase("push-halo", halo_cells)
        c.syncs_device += 1
        c.phase("device-sync", 0)
        c.phase("swap", 0)
        c.gm_loads += halo_cells
        c.gm_halo_loads += halo_cells
        c.phase("pull-halo", halo_cells)
        c.syncs_block += len(regions)
        c.phase("block-sync", 0)
        c.halo_transactions += posed_tx if transpose_halo else raw_tx
    stored = prod(chi - clo for clo, chi in tile_core)
    c.gm_stores += stored
    c.cells_valid += stored * t
    c.phase("store", stored)


def _resident_lazy(c, extents, rad, t, loaded, tile_core, grid_shape, shared_pc, reg_pc):
    """device.py:214-261."""
    per_axis = [even_split(lo, hi, g) for (lo, hi), g in zip(loaded, grid_shape)]
    computed = 0
    for region in itertools.product(*per_axis):
        work = [(max(llo, lo - rad * t), min(lhi, hi + rad * t))
                for (lo, hi), (llo, lhi) in zip(region, loaded)]
        size = prod(hi - lo for lo, hi in work)
        c.gm_loads += size
        c.charge(size * t, shared_pc, reg_pc)
        computed += size * t
        c.syncs_block += t
        store = [(max(clo, lo), min(chi, hi)) for (lo, hi), (clo, chi) in zip(region, tile_core)]
        if all(hi > lo for lo, hi in store):
            stored = prod(hi - lo for lo, hi in store)
            c.gm_stores += stored
            c.cells_valid += stored * t
    c.phase("update", computed)
    c.syncs_device += 1
    c.phase("device-sync", 0)


def reference_counters(offsets, dims: int, extents, params) -> Counters:
    """Dispatch on ``params.scheme`` (planner._ENGINES, planner.py:219)."""
    extents = tuple(int(n) for n in extents)
    offsets = [tuple(int(v) for v in o) for o in offsets]
    if params.scheme == SM_TILING:
        return sm_trace(offsets, dims, extents, params)
    if params.scheme == DEVICE_TILING:
        return device_trace(offsets, dims, extents, params)
    raise ValueError(f"unknown scheme {params.scheme!r}")
