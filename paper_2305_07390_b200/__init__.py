"""B200-native iterated Jacobi sweep (EBISU temporal blocking, arXiv 2305.07390).

Drop-in for the hot path of the reference ``stencilplan`` package: the
stencil spec (``StencilShape``, ``make_benchmark``), grids (``Grid``,
``random_grid``), the sweep (``reference_run`` / ``reference_step``) and the
engine registry (``run_sm_tiling`` / ``run_device_tiling``), executed by
hand-written sm_100a kernels in ``libebisu.so`` through a C ABI
(``include/ebisu.h``).
"""

from .engine import (
    DEVICE_TILING,
    ENGINES,
    SM_TILING,
    ExecutionTrace,
    ParamError,
    TilingParams,
    run_device_tiling,
    run_sm_tiling,
    trace_summary,
)
from .grid import Grid, constant_grid, random_grid, reference_run, reference_step, sweep
from .rng import SplitMix64, uniform_array
from .shapes import (
    BENCHMARK_NAMES,
    CatalogError,
    StencilShape,
    get_shape,
    make_benchmark,
    star_shape,
)

__version__ = "0.1.0"

__all__ = [
    "BENCHMARK_NAMES",
    "CatalogError",
    "DEVICE_TILING",
    "ENGINES",
    "ExecutionTrace",
    "Grid",
    "ParamError",
    "SM_TILING",
    "SplitMix64",
    "StencilShape",
    "TilingParams",
    "constant_grid",
    "get_shape",
    "make_benchmark",
    "random_grid",
    "reference_run",
    "reference_step",
    "run_device_tiling",
    "run_sm_tiling",
    "star_shape",
    "sweep",
    "trace_summary",
    "uniform_array",
]
