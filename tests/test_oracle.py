"""The CPU oracle, pinned against the unmodified reference (tests/golden/).

Also restates the reference's own known-answer tests for the path
(pkg/tests/test_grid.py:17-157) against the oracle, so the oracle is trusted
before it judges the GPU.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import sha256, taps_of
from oracle import reference_run, reference_run_threaded, reference_step, uniform_array
from oracle.stencil_oracle import check_compatible
from paper_2305_07390_b200.rng import SplitMix64
from paper_2305_07390_b200.rng import uniform_array as product_uniform
from paper_2305_07390_b200.shapes import BENCHMARK_NAMES, get_shape, make_benchmark


def _taps(rec):
    return [(tuple(o), c) for o, c in rec["taps"]]


def test_golden_cases_bitwise(golden):
    for rec in golden["cases"]:
        if rec["extents"] == [512, 512] or np.prod(rec["extents"]) > 300_000:
            continue  # the big ones run in test_golden_large
        cells = uniform_array(rec["seed"], int(np.prod(rec["extents"]))).reshape(rec["extents"])
        assert sha256(cells) == rec["input_sha256"], rec["id"]
        out = reference_run(cells, _taps(rec), rec["steps"])
        assert sha256(out) == rec["output_sha256"], (rec["id"], rec["name"])


def test_golden_large(golden):
    # includes BASELINE config 1 (j2d5pt 512^2, 100 steps), the parity anchor
    for rec in golden["cases"]:
        if not (rec["extents"] == [512, 512] or np.prod(rec["extents"]) > 300_000):
            continue
        cells = uniform_array(rec["seed"], int(np.prod(rec["extents"]))).reshape(rec["extents"])
        out = reference_run(cells, _taps(rec), rec["steps"])
        assert sha256(out) == rec["output_sha256"], (rec["id"], rec["name"])


def test_golden_small_arrays(golden, golden_arrays):
    for rec in golden["cases"]:
        key = f"case{rec['id']}_out"
        if key not in golden_arrays:
            continue
        cells = uniform_array(rec["seed"], int(np.prod(rec["extents"]))).reshape(rec["extents"])
        out = reference_run(cells, _taps(rec), rec["steps"])
        assert np.array_equal(out, golden_arrays[key])


def test_product_shapes_match_reference_tap_order(golden):
    # The tap ORDER fixes the summation order; the product's builders must
    # reproduce the reference catalog exactly (shapes.py:91-140).
    for name, taps in golden["catalog_taps"].items():
        st = get_shape(name)
        assert [list(o) for o in st.offsets] == [o for o, _ in taps], name
        assert list(st.coefficients) == [c for _, c in taps], name
        assert st.radius == golden["catalog_radius"][name]
    assert set(BENCHMARK_NAMES) <= set(golden["catalog_taps"])


def test_splitmix_draws(golden):
    g = SplitMix64(0xC0FFEE)
    assert [str(g.next_u64()) for _ in range(8)] == golden["splitmix64_C0FFEE_u64"]
    g = SplitMix64(0xC0FFEE)
    assert [g.uniform() for _ in range(8)] == golden["splitmix64_C0FFEE_uniform"]
    # vectorised == scalar, oracle == product generator
    g = SplitMix64(12345)
    scalar = np.array([g.uniform() for _ in range(100)])
    assert np.array_equal(uniform_array(12345, 100), scalar)
    assert np.array_equal(product_uniform(12345, 100), scalar)
    assert np.array_equal(product_uniform(12345, 40, start=60), scalar[60:])


def test_impulse_known_answer(golden):
    st = make_benchmark("j1d3pt", coefficients=[0.25, 0.5, 0.25])
    cells = np.zeros(11)
    cells[5] = 1.0
    out = reference_step(cells, taps_of(st))
    expected = np.zeros(11)
    expected[4:7] = [0.25, 0.5, 0.25]
    assert np.array_equal(out, expected)
    assert out.tolist() == golden["impulse_j1d3pt"]


def _double_loop_2d5pt(cells, coeffs):
    a, b, c, d, e = coeffs
    n, m = cells.shape
    out = cells.copy()
    for i in range(1, n - 1):
        for j in range(1, m - 1):
            acc = a * cells[i - 1][j]
            acc += b * cells[i][j]
            acc += c * cells[i + 1][j]
            acc += d * cells[i][j - 1]
            acc += e * cells[i][j + 1]
            out[i][j] = acc
    return out


def test_scalar_transcription_2d5pt():
    # reference pkg/tests/test_grid.py:43-66
    st = make_benchmark("j2d5pt")
    cells = uniform_array(42, 256).reshape(16, 16)
    assert np.array_equal(reference_step(cells, taps_of(st)),
                          _double_loop_2d5pt(cells, st.coefficients))


def test_brute_force_3d():
    # reference pkg/tests/test_grid.py:69-91
    st = make_benchmark("j3d7pt")
    cur = uniform_array(7, 12 ** 3).reshape(12, 12, 12)
    expect = cur.copy()
    for _ in range(3):
        new = expect.copy()
        for i in range(1, 11):
            for j in range(1, 11):
                for k in range(1, 11):
                    acc = None
                    for (di, dj, dk), c in st.taps:
                        term = c * expect[i + di][j + dj][k + dk]
                        acc = term if acc is None else acc + term
                    new[i][j][k] = acc
        expect = new
    assert np.array_equal(reference_run(cur, taps_of(st), 3), expect)


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_threaded_oracle_is_bitwise(threads):
    for name, ext, t in (("j2d5pt", (67, 45), 5), ("j2d25pt", (40, 33), 3),
                         ("j3d7pt", (20, 18, 16), 4), ("j1d3pt", (90,), 6)):
        st = get_shape(name)
        cells = uniform_array(7, int(np.prod(ext))).reshape(ext)
        a = reference_run(cells, taps_of(st), t)
        b = reference_run_threaded(cells, taps_of(st), t, threads)
        assert np.array_equal(a, b), (name, threads)


def test_oracle_errors():
    st = make_benchmark("j2d9pt")
    with pytest.raises(ValueError, match="too small"):
        check_compatible(np.zeros((4, 10)), taps_of(st))
    with pytest.raises(ValueError, match="2-D"):
        check_compatible(np.zeros(10), taps_of(st))
    with pytest.raises(ValueError, match=">= 0"):
        reference_run(np.zeros((9, 9)), taps_of(st), -1)


def test_composition_property():
    st = make_benchmark("j2d5pt")
    cells = uniform_array(3, 81).reshape(9, 9)
    for a in range(4):
        for b in range(4):
            whole = reference_run(cells, taps_of(st), a + b)
            parts = reference_run(reference_run(cells, taps_of(st), a), taps_of(st), b)
            assert np.array_equal(whole, parts)
