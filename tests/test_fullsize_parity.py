"""Every BASELINE config at its real size and step count against the oracle.

``tests/golden/fullsize.json`` holds SHA-256 digests (whole output plus 16
axis-0 chunks) of ``reference_run`` at full size, produced by the C oracle
(``oracle/stencil_oracle.c``, pinned bitwise to the unmodified reference by
tests/test_oracle.py) with ``tests/golden/make_fullsize_golden.py``;
``fullsize_samples.npz`` holds the oracle's values at 4096 fixed cells.

Bar (north_star): bitwise in exact mode; within 1e-12 of max |ref| in FMA
mode; within 1e-5 of max |ref| in fp32 mode.  Inputs are generated in HBM
(``ebisu_random_grid_device``, bit-identical to random_grid seed 1).
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2305_07390_b200 as eb
from conftest import GOLDEN_DIR
from paper_2305_07390_b200 import _native, device

pytestmark = pytest.mark.gpu

FMA_RTOL = 1e-12
FP32_RTOL = 1e-5

with open(os.path.join(GOLDEN_DIR, "fullsize.json")) as _f:
    FULL = json.load(_f)
SAMPLES = dict(np.load(os.path.join(GOLDEN_DIR, "fullsize_samples.npz")))


def _digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def _sample_index(total: int, n: int) -> np.ndarray:
    stride = max(1, total // n)
    return (np.arange(n, dtype=np.int64) * stride + stride // 2) % total


def _run(cid, dtype=None, **kw):
    import torch

    rec = FULL["cases"][cid]
    st = eb.get_shape(rec["stencil"])
    d_in = device.random_grid_device(tuple(rec["extents"]), seed=rec["seed"])
    if dtype is not None:
        d_in = d_in.to(dtype)
    out, tr = device.sweep_device(d_in, st, rec["steps"], trace=True, **kw)
    host = out.cpu().numpy()
    del d_in, out
    torch.cuda.empty_cache()
    return rec, host, tr


def _assert_digest(cid, host, tr):
    rec = FULL["cases"][cid]
    got = _digest(host)
    if got != rec["sha256"]:
        b = rec["chunk_rows"]
        bad = [f"rows [{b[i]}, {b[i + 1]})" for i in range(len(b) - 1)
               if _digest(host[b[i]:b[i + 1]]) != rec["chunk_sha256"][i]]
        pytest.fail(f"{cid}: output differs from the oracle in {bad} (kernel {tr['kernel']}, "
                    f"t={tr['t_used']})")


def test_fixture_covers_every_baseline_config():
    ids = set(FULL["cases"])
    assert {"c2_j2d5pt_8192_T1000", "c3_j2d13pt_8192_T96", "c3_j2ds25pt_8192_T96",
            "c4_j3d7pt_512_T500", "c4_j3d27pt_512_T500", "c5_j3d7pt_1024_T100"} <= ids


def test_config2_headline_bitwise():
    """j2d5pt 8192^2 x 1000, the bench workload (default depth 8, persistent)."""
    rec, host, tr = _run("c2_j2d5pt_8192_T1000")
    assert tr["kernel"] == "stream2d_tb"
    _assert_digest("c2_j2d5pt_8192_T1000", host, tr)


@pytest.mark.parametrize("t", [4, 12, 16])
def test_config2_other_depths_bitwise(t):
    rec, host, tr = _run("c2_j2d5pt_8192_T1000", t=t)
    _assert_digest("c2_j2d5pt_8192_T1000", host, tr)


@pytest.mark.parametrize("cid,depths", [("c3_j2d13pt_8192_T96", (2, 3)),
                                        ("c3_j2ds25pt_8192_T96", (1, 2))])
@pytest.mark.parametrize("scheme", ["sm", "device"])
def test_config3_both_schemes_bitwise(cid, depths, scheme):
    code = _native.SCHEME_SM_TILING if scheme == "sm" else _native.SCHEME_DEVICE_TILING
    for t in depths:
        rec, host, tr = _run(cid, t=t, scheme=code)
        _assert_digest(cid, host, tr)


@pytest.mark.parametrize("t", [0, 1, 2, 3, 4])
def test_config4_j3d7pt_bitwise(t):
    rec, host, tr = _run("c4_j3d7pt_512_T500", t=t)
    assert tr["kernel"] == "stream3d_tb"
    _assert_digest("c4_j3d7pt_512_T500", host, tr)


def test_config4_j3d27pt_bitwise():
    rec, host, tr = _run("c4_j3d27pt_512_T500")
    assert tr["kernel"] == "stream3d_tb"
    _assert_digest("c4_j3d27pt_512_T500", host, tr)


def test_config5_1024_cubed_bitwise():
    rec, host, tr = _run("c5_j3d7pt_1024_T100")
    _assert_digest("c5_j3d7pt_1024_T100", host, tr)


def test_odd_width_8191_bitwise():
    if "odd_j2d5pt_8191_T1000" not in FULL["cases"]:
        pytest.skip("fixture not generated")
    rec, host, tr = _run("odd_j2d5pt_8191_T1000")
    _assert_digest("odd_j2d5pt_8191_T1000", host, tr)


def _samples_close(cid, host, rtol):
    ref = SAMPLES[cid]
    got = host.reshape(-1)[_sample_index(host.size, ref.size)].astype(np.float64)
    err = float(np.max(np.abs(got - ref)))
    bound = rtol * float(np.max(np.abs(ref)))
    assert err <= bound, (cid, err, bound)
    return err


@pytest.mark.parametrize("cid", ["c2_j2d5pt_8192_T1000", "c4_j3d7pt_512_T500",
                                 "c4_j3d27pt_512_T500"])
def test_fp32_mode_within_1e5_at_full_size(cid):
    import torch

    rec, host, tr = _run(cid, dtype=torch.float32)
    _samples_close(cid, host, FP32_RTOL)


@pytest.mark.parametrize("cid", ["c2_j2d5pt_8192_T1000", "c4_j3d27pt_512_T500"])
def test_fma_mode_within_1e12_at_full_size(cid):
    rec, host, tr = _run(cid, exact=False)
    _samples_close(cid, host, FMA_RTOL)
