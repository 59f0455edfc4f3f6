"""Full-size golden digests for every BASELINE config, from the C oracle.

Run in the build container (minutes on 8 host threads; needs ~26 GB RAM for
the 1024^3 case):

    python tests/golden/make_fullsize_golden.py [case-id ...]

The C oracle (``oracle/stencil_oracle.c``) is the restatement of the
reference sweep that ``tests/test_oracle.py`` pins bitwise against the 19
digests produced by the UNMODIFIED reference (``make_golden.py``); at these
sizes the numpy reference itself would need hours.  For each case this
writes into ``fullsize.json``: the SHA-256 of the whole ``reference_run``
output (C order, little-endian float64), per-chunk digests along axis 0 (so
a failing GPU test says where), the output sum, and into
``fullsize_samples.npz`` the values at a fixed strided sample of cells
(tolerance checks of the fp32 and FMA modes at full size).

Inputs are ``random_grid(extents, seed)`` (SplitMix64, grid.py:56-60) and the
catalog / star tap lists (shapes.py:91-172), exactly as bench.py builds them.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import c_oracle  # noqa: E402

CHUNKS = 16
NSAMPLES = 4096

# (id, stencil, extents, seed, steps) -- BASELINE.json configs 2-5 at their
# real sizes and step counts (config 1 is in golden.json from the reference
# itself), plus an odd-width config-2 grid for the padded-pitch path.
CASES = [
    ("c2_j2d5pt_8192_T1000", "j2d5pt", (8192, 8192), 1, 1000),
    ("c3_j2d13pt_8192_T96", "j2d13pt", (8192, 8192), 1, 96),
    ("c3_j2ds25pt_8192_T96", "j2ds25pt", (8192, 8192), 1, 96),
    ("c4_j3d7pt_512_T500", "j3d7pt", (512, 512, 512), 1, 500),
    ("c4_j3d27pt_512_T500", "j3d27pt", (512, 512, 512), 1, 500),
    ("c5_j3d7pt_1024_T100", "j3d7pt", (1024, 1024, 1024), 1, 100),
    ("odd_j2d5pt_8191_T1000", "j2d5pt", (8191, 8191), 1, 1000),
]


def taps_of(name: str):
    from paper_2305_07390_b200.shapes import get_shape

    st = get_shape(name)
    return [(tuple(o), float(c)) for o, c in st.taps]


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def chunk_bounds(n0: int):
    return [n0 * i // CHUNKS for i in range(CHUNKS + 1)]


def sample_index(total: int) -> np.ndarray:
    """Fixed strided flat indices (deterministic, spans the whole grid)."""
    stride = max(1, total // NSAMPLES)
    return (np.arange(NSAMPLES, dtype=np.int64) * stride + stride // 2) % total


def main(ids):
    out_json = os.path.join(HERE, "fullsize.json")
    out_npz = os.path.join(HERE, "fullsize_samples.npz")
    doc = json.load(open(out_json)) if os.path.exists(out_json) else {"cases": {}}
    samples = dict(np.load(out_npz)) if os.path.exists(out_npz) else {}
    doc["generator"] = ("tests/golden/make_fullsize_golden.py (C oracle, pinned to the "
                        "reference by tests/test_oracle.py)")
    doc["chunks"] = CHUNKS
    for cid, name, ext, seed, steps in CASES:
        if ids and cid not in ids:
            continue
        t0 = time.time()
        total = int(np.prod(ext))
        cells = c_oracle.uniform_array(seed, total).reshape(ext)
        out = c_oracle.reference_run(cells, taps_of(name), steps)
        del cells
        b = chunk_bounds(ext[0])
        idx = sample_index(total)
        doc["cases"][cid] = {
            "stencil": name, "extents": list(ext), "seed": seed, "steps": steps,
            "sha256": digest(out),
            "chunk_sha256": [digest(out[b[i]:b[i + 1]]) for i in range(CHUNKS)],
            "chunk_rows": b,
            "sum": float(out.sum(dtype=np.float64)),
            "oracle_seconds": round(time.time() - t0, 1),
            "oracle_threads": c_oracle.threads(),
        }
        samples[cid] = out.reshape(-1)[idx].copy()
        del out
        json.dump(doc, open(out_json, "w"), indent=1, sort_keys=True)
        np.savez_compressed(out_npz, **samples)
        print(cid, doc["cases"][cid]["sha256"][:16], f"{time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main(set(sys.argv[1:]))
