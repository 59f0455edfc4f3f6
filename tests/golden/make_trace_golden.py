"""Golden ExecutionTrace counters from the UNMODIFIED reference engines.

Run in the build container (the reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_trace_golden.py

Runs ``stencilplan.engine.run_sm_tiling`` / ``run_device_tiling`` on the
reference's own randomized case generators (``tests/conftest.py:21-80``:
``sm_case``, ``device_case``) for every catalog shape, both schemes and every
lazy / rst / prefetch / transpose_halo combination, plus a few larger
hand-picked geometries (non-dividing last block, multi-tile device grids, a
phase log past the 4096-entry cap), and writes every trace counter to
``traces.json``.  ``tests/test_accounting.py`` checks
``paper_2305_07390_b200.accounting`` against it.
"""

from __future__ import annotations

import hashlib
import itertools
import json
import os

from conftest import device_case, sm_case  # reference tests/conftest.py
from stencilplan import make_benchmark, random_grid
from stencilplan.engine import (
    DEVICE_TILING,
    SM_TILING,
    TilingParams,
    run_device_tiling,
    run_sm_tiling,
)
from stencilplan.rng import SplitMix64
from stencilplan.shapes import BENCHMARK_NAMES

HERE = os.path.dirname(os.path.abspath(__file__))
ENGINES = {SM_TILING: run_sm_tiling, DEVICE_TILING: run_device_tiling}


def phases_digest(phases) -> str:
    return hashlib.sha256(json.dumps([[t, n] for t, n in phases]).encode()).hexdigest()


def record(name, domain, params, trace):
    d = trace.to_dict()
    return {
        "stencil": name, "extents": list(domain),
        "params": {"scheme": params.scheme, "t": params.t, "tile": list(params.tile),
                   "device_tile_grid": list(params.device_tile_grid)
                   if params.device_tile_grid else None,
                   "lazy": params.lazy, "rst": params.rst, "prefetch": params.prefetch,
                   "transpose_halo": params.transpose_halo},
        "counters": {k: d[k] for k in ("gm_loads", "gm_stores", "gm_halo_loads",
                                       "gm_halo_stores", "cells_computed", "cells_valid",
                                       "device_tiles", "halo_transactions")},
        "syncs": d["syncs"],
        "onchip_shared": [trace.onchip_shared.numerator, trace.onchip_shared.denominator],
        "onchip_register": [trace.onchip_register.numerator, trace.onchip_register.denominator],
        "phases_len": len(d["wall_phases"]),
        "phases_sha256": phases_digest(d["wall_phases"]),
        "phases_head": d["wall_phases"][:6],
    }


def main():
    rng = SplitMix64(0x7ACE)
    cases = []
    for name in BENCHMARK_NAMES:
        st = make_benchmark(name)
        for scheme in (SM_TILING, DEVICE_TILING):
            for _ in range(3):
                t = rng.randint(1, 3)
                gen = sm_case if scheme == SM_TILING else device_case
                params, domain = gen(st, rng, t)
                grid = random_grid(domain, seed=rng.next_u64())
                for lazy, rst, pf, th in itertools.product((False, True), repeat=4):
                    params.lazy, params.rst = lazy, rst
                    params.prefetch, params.transpose_halo = pf, th
                    _, tr = ENGINES[scheme](grid, st, params)
                    cases.append(record(name, domain, params, tr))
    extra = [
        ("j2d5pt", (96, 1024), TilingParams(scheme=SM_TILING, t=7, tile=(256,))),
        ("j2d5pt", (20, 30), TilingParams(scheme=SM_TILING, t=1, tile=(30,))),
        ("j3d7pt", (10, 58, 30), TilingParams(scheme=SM_TILING, t=3, tile=(34, 34))),
        ("j3d27pt", (20, 37, 41), TilingParams(scheme=SM_TILING, t=2, tile=(12, 16))),
        ("j1d3pt", (97,), TilingParams(scheme=SM_TILING, t=3, tile=(17,))),
        ("j1d3pt", (97,), TilingParams(scheme=DEVICE_TILING, t=3, tile=(10,),
                                       device_tile_grid=(2,))),
        ("j2d9pt", (60, 70), TilingParams(scheme=DEVICE_TILING, t=2, tile=(10, 12),
                                          device_tile_grid=(2, 2))),
        ("j3d7pt", (40, 50, 46), TilingParams(scheme=DEVICE_TILING, t=2, tile=(10, 10),
                                              device_tile_grid=(2, 2))),
        ("j3d7pt", (600, 20, 22), TilingParams(scheme=DEVICE_TILING, t=3, tile=(9, 10),
                                               device_tile_grid=(2, 2))),
    ]
    for name, domain, params in extra:
        st = make_benchmark(name)
        grid = random_grid(domain, seed=5)
        for lazy in (False, True):
            params.lazy = lazy
            _, tr = ENGINES[params.scheme](grid, st, params)
            cases.append(record(name, domain, params, tr))
    doc = {"generator": "tests/golden/make_trace_golden.py (unmodified reference engines)",
           "cases": cases}
    with open(os.path.join(HERE, "traces.json"), "w") as f:
        json.dump(doc, f, sort_keys=True, separators=(",", ":"))
    print(len(cases), "trace cases")


if __name__ == "__main__":
    main()
