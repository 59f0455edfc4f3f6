"""Generate the golden fixtures from the UNMODIFIED reference.

Run in the build container (the reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports ``stencilplan`` read-only and writes, next to this script:

* ``golden.json`` -- per case: stencil taps (offsets + coefficients, catalog
  order), extents, seed, steps, SHA-256 of the ``reference_run`` output bytes
  (C order, little-endian float64), plus the input digest and a few sampled
  cells; the reference's tap lists for every catalog shape; SplitMix64 draws.
* ``small_cases.npz`` -- full output arrays of the small cases.

Nothing here is imported by the product; tests compare the oracle and the
CUDA path against these files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

import stencilplan  # noqa: F401  (from /root/reference/pkg/src via PYTHONPATH)
from stencilplan import make_benchmark, random_grid, reference_run
from stencilplan.rng import SplitMix64
from stencilplan.shapes import BENCHMARK_NAMES, StencilShape, _star

HERE = os.path.dirname(os.path.abspath(__file__))


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def star(rad: int, name: str) -> StencilShape:
    offs = _star(2, rad)
    n = len(offs)
    return StencilShape(
        name=name, dims=2, taps=tuple((o, 1.0 / n) for o in offs),
        flops_per_cell=2 * n, gm_accesses_per_cell=2,
        sm_accesses_no_rst=n + 1, sm_accesses_with_rst=float(n + 1),
    )


def shape(name: str) -> StencilShape:
    if name == "j2d13pt":
        return star(3, name)
    if name == "j2ds25pt":
        return star(6, name)
    return make_benchmark(name)


# (name, extents, seed, steps, keep_array)
CASES = [
    ("j2d5pt", (512, 512), 1, 100, False),          # BASELINE config 1 (the anchor)
    ("j2d5pt", (16, 16), 42, 1, True),              # test_grid.py:43-66 geometry
    ("j3d7pt", (12, 12, 12), 7, 3, True),           # test_grid.py:69-91 geometry
    ("j3d7pt", (64, 64, 64), 1, 16, False),
    ("j2d5pt", (96, 1024), 3, 7, False),            # test_engine_sm.py:20-27 geometry
    ("j2d5pt", (37, 131), 5, 23, True),             # ragged extents, odd width
    ("j2d5pt", (3, 3), 6, 4, True),                 # smallest legal grid
    ("j1d3pt", (101,), 8, 9, True),
    ("j2d9pt", (40, 66), 9, 5, True),
    ("j2d9pt-gol", (33, 48), 10, 6, True),
    ("j2d25pt", (30, 50), 11, 4, True),
    ("j3d13pt", (14, 18, 22), 12, 3, True),
    ("j3d17pt", (11, 20, 24), 13, 4, True),
    ("j3d27pt", (10, 16, 18), 14, 5, True),
    ("poisson", (12, 15, 20), 15, 3, True),
    ("j2d13pt", (40, 64), 16, 3, True),
    ("j2ds25pt", (50, 72), 17, 3, True),
    ("j3d27pt", (32, 40, 48), 18, 8, False),
    ("j2d5pt", (200, 260), 19, 50, False),
]


def main():
    cases = []
    arrays = {}
    for i, (name, ext, seed, steps, keep) in enumerate(CASES):
        st = shape(name)
        g = random_grid(ext, seed)
        out = reference_run(g, st, steps).cells
        rec = {
            "id": i,
            "name": name,
            "extents": list(ext),
            "seed": seed,
            "steps": steps,
            "taps": [[list(o), c] for o, c in st.taps],
            "input_sha256": digest(g.cells),
            "output_sha256": digest(out),
            "output_sum": float(out.sum()),
            "samples": [[list(map(int, idx)), float(out[idx])]
                        for idx in [tuple(n // 2 for n in ext), tuple(1 for _ in ext),
                                    tuple(n - 2 for n in ext)]],
        }
        cases.append(rec)
        if keep:
            arrays[f"case{i}_out"] = out
        print(f"case {i}: {name} {ext} T={steps} -> {rec['output_sha256'][:16]}", file=sys.stderr)

    catalog = {n: [[list(o), c] for o, c in shape(n).taps]
               for n in list(BENCHMARK_NAMES) + ["j2d13pt", "j2ds25pt"]}
    catalog_radius = {n: shape(n).radius for n in catalog}

    rng = SplitMix64(0xC0FFEE)
    draws = [str(rng.next_u64()) for _ in range(8)]
    rng = SplitMix64(0xC0FFEE)
    uniforms = [rng.uniform() for _ in range(8)]

    # Known answers from the reference's own tests (pkg/tests/test_grid.py).
    impulse = reference_run(
        stencilplan.grid.Grid(np.eye(1, 11, 5).ravel()),
        make_benchmark("j1d3pt", coefficients=[0.25, 0.5, 0.25]), 1).cells

    doc = {
        "generator": "tests/golden/make_golden.py (unmodified reference stencilplan, "
                     "pkg/src/stencilplan/grid.py:106 reference_run)",
        "numpy": np.__version__,
        "cases": cases,
        "catalog_taps": catalog,
        "catalog_radius": catalog_radius,
        "splitmix64_C0FFEE_u64": draws,
        "splitmix64_C0FFEE_uniform": uniforms,
        "impulse_j1d3pt": impulse.tolist(),
    }
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(doc, f, indent=1, sort_keys=True)
        f.write("\n")
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **arrays)


if __name__ == "__main__":
    main()
