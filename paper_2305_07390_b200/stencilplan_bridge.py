"""Register the B200 engines inside an unmodified ``stencilplan`` install.

This is the reference-side binding a ``stencilplan`` maintainer adds to make
the B200 sweep the engine behind the reference's own API:

    import stencilplan
    from paper_2305_07390_b200 import stencilplan_bridge
    stencilplan_bridge.install(stencilplan)          # engines -> B200
    stencilplan_bridge.install(stencilplan, reference_run=True)   # + the oracle

``install`` swaps the engine registry the planner dispatches on
(``planner._ENGINES``, planner.py:219 -> ``_simulate_one`` :222-251 -> CLI
``simulate`` cli.py:106 and HTTP ``POST /simulate`` service.py:102-107) and
the module attributes callers import (``stencilplan.engine.run_sm_tiling`` /
``run_device_tiling``, engine/__init__.py:3-7), optionally also
``stencilplan.reference_run`` / ``reference_step`` (grid.py:96-113; the
planner's own oracle call, planner.py:228, is left on numpy).

Each B200 engine takes and returns the reference's own types: a
``stencilplan.grid.Grid`` in, ``(stencilplan.grid.Grid,
stencilplan.engine.ExecutionTrace)`` out, with the counters the reference
engine would have produced (``accounting.py``) and the GPU facts of the
real run in ``trace.b200``; invalid parameters raise the reference's
``stencilplan.engine.ParamError`` with the reference's messages.  The sweep
itself runs only on the GPU (``libebisu.so``); there is no CPU fallback.
"""

from __future__ import annotations

from . import engine as _engine
from .grid import Grid as _Grid
from .grid import sweep as _sweep

_SAVED: dict = {}
ENGINE_CALLS: dict = {}  # scheme -> B200 engine invocations in this process


def _to_params(params):
    return _engine.TilingParams(
        scheme=params.scheme, t=params.t, tile=tuple(params.tile),
        device_tile_grid=tuple(params.device_tile_grid)
        if params.device_tile_grid is not None else None,
        lazy=bool(params.lazy), rst=bool(params.rst), prefetch=bool(params.prefetch),
        transpose_halo=bool(params.transpose_halo), queue_variant=params.queue_variant,
        workers=int(params.workers))


def _to_ref_trace(sp, tr):
    out = sp.engine.ExecutionTrace()
    for f in ("gm_loads", "gm_stores", "gm_halo_loads", "gm_halo_stores", "onchip_shared",
              "onchip_register", "syncs_block", "syncs_device", "cells_computed",
              "cells_valid", "device_tiles", "halo_transactions"):
        setattr(out, f, getattr(tr, f))
    out.wall_phases = list(tr.wall_phases)
    # what actually ran on the GPU (not a reference field; to_dict ignores it)
    out.b200 = dict(tr.gpu, kernel=tr.kernel, t_used=tr.t_used, elapsed_ms=tr.elapsed_ms,
                    kernel_launches=tr.kernel_launches)
    return out


def make_engine(sp, scheme: str):
    """B200 engine for ``scheme`` speaking the types of the ``stencilplan``
    module ``sp`` (the ``planner._ENGINES`` signature)."""
    fn = _engine.ENGINES[scheme]

    def b200_engine(grid, stencil, params):
        ENGINE_CALLS[scheme] = ENGINE_CALLS.get(scheme, 0) + 1
        try:
            p = _to_params(params)
            out, tr = fn(_Grid(grid.cells, grid.boundary), stencil, p)
        except _engine.ParamError as exc:
            raise sp.engine.ParamError(str(exc)) from None
        return sp.grid.Grid(out.cells, grid.boundary), _to_ref_trace(sp, tr)

    b200_engine.__name__ = fn.__name__
    b200_engine.__qualname__ = fn.__name__
    b200_engine.__doc__ = f"B200 {scheme} engine (libebisu.so) in stencilplan types"
    return b200_engine


def make_reference_run(sp):
    def reference_run(grid, stencil, t: int):
        if t < 0:
            raise ValueError("step count must be >= 0")
        out = _sweep(_Grid(grid.cells, grid.boundary), stencil, t)
        return sp.grid.Grid(out.cells.copy() if t == 0 else out.cells, grid.boundary)

    def reference_step(grid, stencil):
        return reference_run(grid, stencil, 1)

    return reference_run, reference_step


def install(sp=None, engines: bool = True, reference_run: bool = False):
    """Point ``stencilplan`` (module ``sp``, default: ``import stencilplan``)
    at the B200 path.  Idempotent; ``uninstall`` restores the originals."""
    if sp is None:
        import stencilplan as sp  # noqa: PLC0415
    import stencilplan.engine.device  # noqa: F401,PLC0415
    import stencilplan.engine.sm  # noqa: F401,PLC0415
    import stencilplan.planner  # noqa: F401,PLC0415

    def swap(mod, name, value):
        key = (mod.__name__, name)
        if key not in _SAVED:
            _SAVED[key] = (mod, getattr(mod, name))
        setattr(mod, name, value)

    if engines:
        sm = make_engine(sp, _engine.SM_TILING)
        dev = make_engine(sp, _engine.DEVICE_TILING)
        reg = dict(sp.planner._ENGINES)
        reg[_engine.SM_TILING] = sm
        reg[_engine.DEVICE_TILING] = dev
        swap(sp.planner, "_ENGINES", reg)
        swap(sp.engine, "run_sm_tiling", sm)
        swap(sp.engine, "run_device_tiling", dev)
        swap(sp.engine.sm, "run_sm_tiling", sm)
        swap(sp.engine.device, "run_device_tiling", dev)
    if reference_run:
        run, step = make_reference_run(sp)
        # (planner.reference_run stays the numpy oracle: _simulate_one's
        # parity check keeps comparing against the reference arithmetic)
        for mod in (sp, sp.grid):
            swap(mod, "reference_run", run)
        for mod in (sp, sp.grid):
            swap(mod, "reference_step", step)
    return sp


def uninstall():
    for (_, name), (mod, value) in list(_SAVED.items()):
        setattr(mod, name, value)
    _SAVED.clear()


def main(argv=None) -> int:
    """``stencilplan`` CLI with the B200 engines -- SURVEY §8(f)4's
    ``stencilplan simulate --engine b200``:

        python -m paper_2305_07390_b200.stencilplan_bridge simulate --suite s.json

    installs the engines into the unmodified reference package, then hands
    ``argv`` to the reference's own front end (cli.py:69-123): ``simulate``
    runs every suite case through ``planner._simulate_one`` on the GPU and
    checks it against the reference's numpy ``reference_run`` (exit 1 on a
    mismatch), ``plan`` / ``validate`` / ``report`` / ``catalog`` / ``serve``
    behave as in the reference (``serve``: HTTP ``POST /simulate`` on the
    GPU engines)."""
    import sys

    import stencilplan.cli  # noqa: PLC0415

    install()
    rc = stencilplan.cli.main(sys.argv[1:] if argv is None else argv)
    print(f"[b200] engine calls: {sum(ENGINE_CALLS.values())} {ENGINE_CALLS}", file=sys.stderr)
    return rc


if __name__ == "__main__":
    raise SystemExit(main())
