"""GPU parity: the sm_100a path through the C ABI vs the oracle / golden
fixtures.  Bar: bitwise in exact mode (IEEE binary64 mul/add in tap order),
1e-12 relative (of max |ref|) in FMA mode.  (north_star tolerance: 1e-12 fp64.)
"""

from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2305_07390_b200 as eb
from conftest import sha256, taps_of
from oracle import reference_run as oracle_run
from oracle import reference_run_threaded
from paper_2305_07390_b200 import _native

pytestmark = pytest.mark.gpu

FMA_RTOL = 1e-12


def _shape(name):
    return eb.get_shape(name)


def test_library_is_the_native_one():
    lib = _native.load()
    assert lib.ebisu_device_count() >= 1
    assert os.path.samefile(lib._name, _native.LIB_PATH)


def test_golden_cases_bitwise_auto(golden):
    for rec in golden["cases"]:
        st = _shape(rec["name"])
        g = eb.random_grid(rec["extents"], rec["seed"])
        out, tr = eb.sweep(g, st, rec["steps"], trace=True)
        assert sha256(out.cells) == rec["output_sha256"], (rec["id"], rec["name"], tr)


@pytest.mark.parametrize("t", list(range(1, 17)))
def test_j2d5pt_every_depth_bitwise(golden, t):
    # BASELINE config 1 (512^2, 100 steps) and a ragged 200x260 case, every fused depth
    for rec in golden["cases"]:
        if rec["name"] != "j2d5pt" or rec["extents"] not in ([512, 512], [200, 260],
                                                             [96, 1024]):
            continue
        g = eb.random_grid(rec["extents"], rec["seed"])
        for persistent in (True, False):
            out, tr = eb.sweep(g, _shape("j2d5pt"), rec["steps"], t=t, persistent=persistent,
                               trace=True)
            assert tr["kernel"] == "stream2d_tb", tr
            assert sha256(out.cells) == rec["output_sha256"], (rec["id"], t, persistent)


CASES_2D = {
    "j2d5pt": list(range(1, 17)),
    "j2d9pt-gol": [1, 2, 3, 4, 6, 8],
    "j2d9pt": [1, 2, 3, 4, 5],
    "j2d25pt": [1, 2, 3, 4],
    "j2d13pt": [1, 2, 3],
    "j2ds25pt": [1, 2],
}


@pytest.mark.parametrize("name", list(CASES_2D))
def test_2d_shapes_all_depths_ragged(name):
    st = _shape(name)
    rng = eb.SplitMix64(hash(name) & 0xFFFF)
    for t in CASES_2D[name]:
        for _ in range(3):
            n0 = 2 * st.radius + 1 + rng.randint(0, 300)
            n1 = 2 * (st.radius + 1 + rng.randint(0, 400) // 2)  # even width -> TMA path
            steps = rng.randint(1, 3 * t + 2)
            g = eb.random_grid((n0, n1), rng.next_u64())
            ref = oracle_run(g.cells, taps_of(st), steps)
            out, tr = eb.sweep(g, st, steps, t=t, trace=True)
            assert np.array_equal(out.cells, ref), (name, t, (n0, n1), steps, tr)


def test_odd_width_runs_padded_tb_and_generic_shapes_run_resident_or_naive():
    # odd row pitch (TMA needs 16-byte strides): the TB kernel runs on
    # row-padded copies; every depth, both schemes, fp64 + fp32 layouts
    st = _shape("j2d5pt")
    for ext, steps in (((37, 131), 23), ((200, 257), 50), ((64, 1023), 19)):
        g = eb.random_grid(ext, 5)
        ref = oracle_run(g.cells, taps_of(st), steps)
        for t in (0, 1, 3, 8):
            out, tr = eb.sweep(g, st, steps, t=t, trace=True)
            assert tr["kernel"] == "stream2d_tb", (ext, t, tr)
            assert np.array_equal(out.cells, ref), (ext, t)
        out, tr = eb.sweep(g, st, steps, scheme=_native.SCHEME_DEVICE_TILING, trace=True)
        assert tr["kernel"] == "halo2d_tb", tr
        assert np.array_equal(out.cells, ref), ext
        out, tr = eb.sweep(g, st, steps, trace=True, dtype=np.float32)
        assert tr["kernel"] == "stream2d_tb", tr
        assert np.max(np.abs(out.cells - ref)) <= 1e-5 * np.max(np.abs(ref)), ext
    for name in ("j2d9pt", "j2d25pt", "j2ds25pt"):
        st = _shape(name)
        g = eb.random_grid((60, 2 * 128 + 3 * st.radius * 4 + 1), 3)
        out, tr = eb.sweep(g, st, 5, trace=True)
        assert tr["kernel"] == "stream2d_tb", (name, tr)
        assert np.array_equal(out.cells, oracle_run(g.cells, taps_of(st), 5)), name
    # reversed tap order = a different summation order -> generic kernel, still exact
    rev = eb.StencilShape("rev", 2, tuple(reversed(st.taps)), 2 * len(st.taps), 2,
                          len(st.taps) + 1, 4.0)
    g = eb.random_grid((40, 64), 9)
    ref = oracle_run(g.cells, taps_of(rev), 7)
    out, tr = eb.sweep(g, rev, 7, trace=True)
    assert tr["kernel"] in ("resident_tb", "naive_step"), tr
    assert np.array_equal(out.cells, ref)
    for scheme, kern in ((_native.SCHEME_NAIVE, "naive_step"),
                         (_native.SCHEME_RESIDENT, "resident_tb")):
        out, tr = eb.sweep(g, rev, 7, scheme=scheme, trace=True)
        assert tr["kernel"] == kern, tr
        assert np.array_equal(out.cells, ref), kern


def test_j1d3pt_bitwise_resident_and_naive():
    st = _shape("j1d3pt")
    g = eb.random_grid((301,), 77)
    ref = oracle_run(g.cells, taps_of(st), 6)
    out, tr = eb.sweep(g, st, 6, trace=True)
    assert tr["kernel"] in ("resident_tb", "naive_step"), tr  # planner's cost model
    assert np.array_equal(out.cells, ref)
    out, tr = eb.sweep(g, st, 6, scheme=_native.SCHEME_RESIDENT, trace=True)
    assert tr["kernel"] == "resident_tb", tr
    assert np.array_equal(out.cells, ref)
    out, tr = eb.sweep(g, st, 6, scheme=_native.SCHEME_NAIVE, trace=True)
    assert tr["kernel"] == "naive_step"
    assert np.array_equal(out.cells, ref)


# ---- resident-tile kernel (any tap set, ebisu_generic.cu) ---------------------

def _random_shape(rng, dims, rad):
    """A user stencil the specialised kernels do not cover: random offsets
    within radius `rad` (zero offset included, any order), random coefficients
    (shapes.py:27-56 accepts any such tap set)."""
    import itertools

    box = [o for o in itertools.product(range(-rad, rad + 1), repeat=dims)]
    n = 1 + rng.randint(1, min(len(box) - 1, 12))
    picks = {tuple([0] * dims)}
    edge = tuple([rad] + [0] * (dims - 1))  # the radius is attained
    picks.add(edge)
    while len(picks) < n:
        picks.add(box[rng.randint(0, len(box) - 1)])
    offs = list(picks)
    # shuffle (tap order = summation order)
    for i in range(len(offs) - 1, 0, -1):
        j = rng.randint(0, i)
        offs[i], offs[j] = offs[j], offs[i]
    taps = tuple((o, 0.05 + 0.9 * rng.uniform() / len(offs)) for o in offs)
    return eb.StencilShape("user", dims, taps, 2 * len(taps), 2, len(taps) + 1,
                           float(min(4, len(taps) + 1)))


@pytest.mark.parametrize("dims", [1, 2, 3])
def test_resident_kernel_random_user_stencils_bitwise(dims):
    """Random user tap sets (random offsets, order and coefficients) at every
    depth 1..6 on ragged grids, odd extents included: bitwise equal to the
    oracle (exact mode) and within 1e-12 in FMA mode."""
    rng = eb.SplitMix64(0xC0FFEE + dims)
    for case in range(6):
        rad = 1 + rng.randint(0, 2)
        st = _random_shape(rng, dims, rad)
        if dims == 1:
            ext = (2 * rad + 1 + rng.randint(0, 40000),)
        elif dims == 2:
            ext = (2 * rad + 1 + rng.randint(0, 300), 2 * rad + 1 + rng.randint(0, 300))
        else:
            ext = tuple(2 * rad + 1 + rng.randint(0, 40) for _ in range(3))
        g = eb.random_grid(ext, rng.next_u64())
        steps = rng.randint(1, 13)
        ref = oracle_run(g.cells, taps_of(st), steps)
        for t in (0, 1, 2, 3, 6):
            out, tr = eb.sweep(g, st, steps, t=t, scheme=_native.SCHEME_RESIDENT, trace=True)
            assert tr["kernel"] == "resident_tb", tr
            assert np.array_equal(out.cells, ref), (dims, case, ext, steps, t, st.taps)
        out = eb.sweep(g, st, steps, scheme=_native.SCHEME_RESIDENT, exact=False)
        assert np.max(np.abs(out.cells - ref)) <= FMA_RTOL * np.max(np.abs(ref))
        out = eb.sweep(g, st, steps, scheme=_native.SCHEME_RESIDENT, dtype=np.float32)
        assert np.max(np.abs(out.cells - ref)) <= 1e-5 * np.max(np.abs(ref))


@pytest.mark.parametrize("name", ["j1d3pt", "j2d5pt", "j2d9pt-gol", "j2d13pt", "j2ds25pt",
                                  "j3d7pt", "j3d27pt", "poisson"])
def test_resident_kernel_catalog_shapes_bitwise(name):
    """The resident-tile kernel forced on catalog shapes (the specialised
    kernels' cross-check), golden-size grids, depths 1..4."""
    st = _shape(name)
    r = st.radius
    ext = {1: (50001,), 2: (257, 2 * r + 301), 3: (33, 2 * r + 29, 45)}[st.dims]
    g = eb.random_grid(ext, 11)
    ref = oracle_run(g.cells, taps_of(st), 9)
    for t in (1, 2, 4):
        out, tr = eb.sweep(g, st, 9, t=t, scheme=_native.SCHEME_RESIDENT, trace=True)
        assert tr["kernel"] == "resident_tb" and tr["t_used"] == t, tr
        assert np.array_equal(out.cells, ref), (name, t)


def test_resident_kernel_output_plane_range():
    """out_planes (the multi-GPU band / interior split) on the resident kernel:
    only planes [lo, hi) are written, and they equal the full sweep's."""
    from paper_2305_07390_b200 import device

    torch = _torch()
    rng = eb.SplitMix64(5)
    st = _random_shape(rng, 2, 2)
    d_in = device.random_grid_device((300, 200), seed=4)
    full = device.sweep_device(d_in, st, 3, params=_native.make_params(
        scheme=_native.SCHEME_RESIDENT, t=3))
    out = torch.full_like(d_in, -7.0)
    prm = _native.make_params(scheme=_native.SCHEME_RESIDENT, t=3, out_planes=(40, 170))
    device.sweep_device(d_in, st, 3, out=out, params=prm)
    assert torch.equal(out[40:170], full[40:170])
    assert bool((out[:40] == -7.0).all()) and bool((out[170:] == -7.0).all())


CASES_3D = {
    "j3d7pt": [1, 2, 3, 4],
    "j3d13pt": [1, 2],
    "j3d17pt": [1, 2],
    "j3d27pt": [1, 2],
    "poisson": [1, 2],
}


@pytest.mark.parametrize("name", list(CASES_3D))
def test_3d_shapes_all_depths_ragged(name):
    st = _shape(name)
    rng = eb.SplitMix64(hash(name) & 0xFFFF)
    r = st.radius
    for t in CASES_3D[name]:
        for _ in range(3):
            n0 = 2 * r + 1 + rng.randint(0, 40)
            n1 = 2 * r + 1 + rng.randint(0, 90)
            n2 = 2 * (r + 1 + rng.randint(0, 90) // 2)  # even: TMA path
            steps = rng.randint(1, 2 * t + 2)
            g = eb.random_grid((n0, n1, n2), rng.next_u64())
            ref = oracle_run(g.cells, taps_of(st), steps)
            out, tr = eb.sweep(g, st, steps, t=t, trace=True)
            assert tr["kernel"] == "stream3d_tb", tr
            assert np.array_equal(out.cells, ref), (name, t, (n0, n1, n2), steps, tr)


def _variants(st, t, ext, steps, scheme=0):
    """Yield (variant, trace, output) for every registered kernel variant."""
    g = eb.random_grid(ext, 97 + t)
    for v in range(64):
        prm = _native.make_params(t=t, variant=v, scheme=scheme)
        try:
            out, tr = eb.sweep(g, st, steps, params=prm, trace=True)
        except Exception as e:  # past the last registered variant
            assert "variant" in str(e), e
            return
        yield g, v, tr, out


@pytest.mark.parametrize("name", list(CASES_3D))
def test_3d_every_registered_variant_bitwise(name):
    st = _shape(name)
    for t in CASES_3D[name]:
        steps = 3 * t + 1
        for ext in ((37, 71, 134), (2 * st.radius + 3, 300, 66)):
            ref = None
            for g, v, tr, out in _variants(st, t, ext, steps):
                if ref is None:
                    ref = oracle_run(g.cells, taps_of(st), steps)
                assert tr["kernel"] == "stream3d_tb", tr
                assert np.array_equal(out.cells, ref), (name, t, v, ext, tr)


def test_3d_lane_variants_and_persistence():
    st = _shape("j3d7pt")
    g = eb.random_grid((40, 70, 134), 11)
    ref = oracle_run(g.cells, taps_of(st), 13)
    for t in (2, 3, 4):
        for persistent in (True, False):
            out = eb.sweep(g, st, 13, t=t, persistent=persistent)
            assert np.array_equal(out.cells, ref), (t, persistent)


def test_3d_odd_last_extent_runs_padded_tb():
    for name in ("j3d7pt", "j3d27pt", "j3d13pt"):
        st = _shape(name)
        for ext in ((17, 19, 23), (20, 45, 71)):
            g = eb.random_grid(ext, 5)
            out, tr = eb.sweep(g, st, 5, trace=True)
            assert tr["kernel"] == "stream3d_tb", (name, ext, tr)
            assert np.array_equal(out.cells, oracle_run(g.cells, taps_of(st), 5)), (name, ext)


def test_full_size_512_cubed_against_oracle():
    # BASELINE config 4 geometry (j3d7pt 512^3): one t=3 epoch + 1 remainder step
    from paper_2305_07390_b200 import device

    torch = _torch()
    st = eb.make_benchmark("j3d7pt")
    d_in = device.random_grid_device((512, 512, 512), seed=1)
    out, tr = device.sweep_device(d_in, st, 4, t=3, trace=True)
    assert tr["kernel"] == "stream3d_tb"
    torch.cuda.synchronize()
    ref = reference_run_threaded(d_in.cpu().numpy(), taps_of(st), 4, os.cpu_count() or 4)
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("name", ["j2d5pt", "j2d25pt", "j3d7pt"])
def test_fma_mode_within_tolerance(name):
    st = _shape(name)
    ext = (130, 258) if st.dims == 2 else (20, 30, 34)
    g = eb.random_grid(ext, 4)
    out = eb.sweep(g, st, 20, exact=False)
    ref = oracle_run(g.cells, taps_of(st), 20)
    err = np.max(np.abs(out.cells - ref))
    assert err <= FMA_RTOL * np.max(np.abs(ref)), err


def test_coefficients_are_runtime():
    st = eb.make_benchmark("j2d5pt", coefficients=[0.1, 0.3, 0.2, 0.25, 0.15])
    g = eb.random_grid((64, 128), 3)
    assert np.array_equal(eb.reference_run(g, st, 9).cells,
                          oracle_run(g.cells, taps_of(st), 9))


PER_TAP_DEPTHS = {"j2d5pt": [1, 2, 4, 8], "j2d9pt-gol": [1, 2, 4, 8], "j2d9pt": [1, 2, 4],
                  "j2d25pt": [1, 2, 3], "j2d13pt": [1, 2, 3], "j2ds25pt": [1, 2],
                  "j3d7pt": [1, 2, 3, 4], "j3d27pt": [1, 2], "j3d13pt": [1, 2],
                  "j3d17pt": [1, 2], "poisson": [1, 2]}


@pytest.mark.parametrize("name", list(PER_TAP_DEPTHS))
def test_per_tap_kernels_bitwise(name):
    """The per-tap kernel family (non-uniform coefficients): forced with
    per_tap_products=1 on the catalog coefficients and selected automatically
    for non-uniform ones -- both bitwise against the oracle."""
    base = _shape(name)
    rng = eb.SplitMix64(7 + len(name))
    coeffs = [0.05 + 0.9 * rng.uniform() / len(base.taps) for _ in base.taps]
    nonuni = base.with_coefficients(coeffs)
    r = base.radius
    ext = (3 * r + 40, 2 * r + 70, 2 * (r + 30)) if base.dims == 3 else (2 * r + 150, 2 * (r + 160))
    g = eb.random_grid(ext[:base.dims], 31)
    for t in PER_TAP_DEPTHS[name]:
        steps = 2 * t + 1
        for st, forced in ((base, True), (nonuni, False)):
            prm = _native.make_params(t=t, per_tap_products=forced)
            out, tr = eb.sweep(g, st, steps, params=prm, trace=True)
            assert tr["kernel"] in ("stream2d_tb", "stream3d_tb", "halo2d_tb"), tr
            ref = oracle_run(g.cells, taps_of(st), steps)
            assert np.array_equal(out.cells, ref), (name, t, forced)
        # FMA chain with non-uniform coefficients: tolerance, not bitwise
        out = eb.sweep(g, nonuni, steps, params=_native.make_params(t=t, exact=False))
        ref = oracle_run(g.cells, taps_of(nonuni), steps)
        assert np.max(np.abs(out.cells - ref)) <= FMA_RTOL * np.max(np.abs(ref)), (name, t)


def test_purity_and_boundary_tag():
    st = eb.make_benchmark("j2d5pt")
    g = eb.Grid(eb.random_grid((10, 10), seed=5).cells, "skip-update")
    before = g.cells.copy()
    out = eb.reference_run(g, st, 3)
    assert np.array_equal(g.cells, before)
    assert out.boundary == "skip-update"


def test_engines_reference_style(rng):
    # reference tests/conftest.py:21-100 case generators, engine vs oracle
    for name in ("j2d5pt", "j2d9pt", "j2d9pt-gol", "j2d25pt", "j1d3pt", "j3d7pt", "j3d27pt"):
        st = eb.make_benchmark(name)
        rad = st.radius
        for _ in range(5):
            t = rng.randint(1, 3)
            core = rng.randint(max(4, rad * 2), 10)
            tile = core + 2 * rad * t
            if st.dims == 1:
                params = eb.TilingParams(scheme=eb.SM_TILING, t=t, tile=(tile,))
                domain = (rng.randint(1, 3) * core + 2 * rad,)
            elif st.dims == 2:
                params = eb.TilingParams(scheme=eb.SM_TILING, t=t, tile=(tile,))
                domain = (2 * rad + rng.randint(6, 14), rng.randint(1, 3) * core + 2 * rad)
            else:
                params = eb.TilingParams(scheme=eb.SM_TILING, t=t, tile=(tile, tile))
                domain = (2 * rad + rng.randint(6, 14), rng.randint(1, 2) * core + 2 * rad,
                          rng.randint(1, 2) * core + 2 * rad)
            g = eb.random_grid(domain, rng.next_u64())
            out, trace = eb.run_sm_tiling(g, st, params)
            assert np.array_equal(out.cells, oracle_run(g.cells, taps_of(st), t)), (name, domain)
            assert trace.cells_valid > 0
            s = eb.trace_summary(trace, st, params, domain)
            assert s.a_gm_measured > 0


# ---- device-resident path at BASELINE sizes -------------------------------------


def _torch():
    import torch

    return torch


def test_device_rng_bit_identical():
    from paper_2305_07390_b200 import device

    d = device.random_grid_device((257, 129), seed=99)
    assert np.array_equal(d.cpu().numpy(), eb.random_grid((257, 129), 99).cells)


def test_full_size_8192_against_oracle():
    # BASELINE config 2 geometry: t=8 epoch + remainder through the 1-step kernel.
    from paper_2305_07390_b200 import device

    torch = _torch()
    st = eb.make_benchmark("j2d5pt")
    steps = 9
    d_in = device.random_grid_device((8192, 8192), seed=1)
    out = device.sweep_device(d_in, st, steps, t=8)
    torch.cuda.synchronize()
    ref = reference_run_threaded(d_in.cpu().numpy(), taps_of(st), steps, os.cpu_count() or 4)
    assert np.array_equal(out.cpu().numpy(), ref)


def test_full_size_composition_and_persistence():
    # size-independent properties at full size: run(16) == run(8) o run(8), and
    # persistent (cooperative, grid.sync) == one launch per epoch, bitwise.
    from paper_2305_07390_b200 import device

    torch = _torch()
    st = eb.make_benchmark("j2d5pt")
    d_in = device.random_grid_device((8192, 8192), seed=2)
    a = device.sweep_device(d_in, st, 48, t=8, persistent=True)
    b = device.sweep_device(d_in, st, 48, t=8, persistent=False)
    h = device.sweep_device(device.sweep_device(d_in, st, 24, t=8), st, 24, t=6)
    torch.cuda.synchronize()
    assert device.compare_device(a, b)["mismatches"] == 0
    assert device.compare_device(a, h)["mismatches"] == 0
    # maximum principle (convex coefficients): values stay in [min, max] of input
    assert float(a.max()) <= float(d_in.max()) and float(a.min()) >= float(d_in.min())


CASES_H2D = {
    "j2d5pt": [4, 6, 8, 12, 16],
    "j2d9pt-gol": [2, 4],
    "j2d9pt": [2, 4],
    "j2d25pt": [2, 3],
    "j2d13pt": [1, 2, 3, 4],
    "j2ds25pt": [1, 2, 3, 4],
}


@pytest.mark.parametrize("name", list(CASES_H2D))
def test_halo_exchange_2d_bitwise(name):
    """device-tiling scheme (CTA strips exchanging per-level edge columns):
    generic strips (n1 < 2 strips), edge-aligned strips (n1 >= 2 strips, the
    frame in the first/last strip), ragged heights, remainders."""
    st = _shape(name)
    rng = eb.SplitMix64(0x4A10 + len(name))
    r = st.radius
    for t in CASES_H2D[name]:
        for n1 in (2 * (r + 1 + rng.randint(0, 300) // 2), 2 * (1100 + rng.randint(0, 700) // 2),
                   2200):
            n0 = 2 * r + 1 + rng.randint(0, 200)
            steps = rng.randint(t, 3 * t + 1)
            g = eb.random_grid((n0, n1), rng.next_u64())
            ref = oracle_run(g.cells, taps_of(st), steps)
            prm = _native.make_params(scheme=_native.SCHEME_DEVICE_TILING, t=t)
            out, tr = eb.sweep(g, st, steps, params=prm, trace=True)
            assert tr["kernel"] == "halo2d_tb", tr
            assert np.array_equal(out.cells, ref), (name, t, (n0, n1), steps)
            if t == CASES_H2D[name][0]:
                prm = _native.make_params(scheme=_native.SCHEME_DEVICE_TILING, t=t,
                                          per_tap_products=True)
                out = eb.sweep(g, st, steps, params=prm)
                assert np.array_equal(out.cells, ref), (name, t, "per-tap")


@pytest.mark.parametrize("name,ext,t,scheme", [
    ("j2d5pt", (300, 258), 8, 0), ("j2d5pt", (300, 2200), 4, 3), ("j2ds25pt", (260, 400), 2, 0),
    ("j3d7pt", (70, 66, 130), 4, 0), ("j3d27pt", (41, 40, 70), 2, 0), ("j3d13pt", (50, 34, 66), 1, 0),
])
def test_output_plane_range(name, ext, t, scheme):
    """ebisu_params.out_planes (the multi-GPU band/interior split): two ranged
    calls tile the full one-epoch result bitwise and nothing outside the range
    is written."""
    from paper_2305_07390_b200 import device

    torch = _torch()
    st = _shape(name)
    d_in = device.random_grid_device(ext, seed=5)
    full = torch.empty_like(d_in)
    device.sweep_device(d_in, st, t, out=full, params=_native.make_params(t=t, scheme=scheme))
    cut = ext[0] // 3 + 1
    split = torch.full_like(d_in, float("nan"))
    for lo, hi in ((cut, ext[0]), (0, cut)):
        prm = _native.make_params(t=t, scheme=scheme, out_planes=(lo, hi))
        device.sweep_device(d_in, st, t, out=split, params=prm)
        if lo == cut:  # first call: nothing below the range written yet
            assert torch.isnan(split[:cut]).all()
    torch.cuda.synchronize()
    assert torch.equal(split, full), (name, ext, t)
    ref = oracle_run(d_in.cpu().numpy(), taps_of(st), t)
    assert np.array_equal(full.cpu().numpy(), ref)
    # a ranged call that would need several epochs is refused
    with pytest.raises(Exception, match="single fused epoch"):
        device.sweep_device(d_in, st, 2 * t + 1, out=split,
                            params=_native.make_params(t=t, out_planes=(0, cut)))



FP32_RTOL = 1e-5  # north_star: fp32 outputs within 1e-5 of the fp64 reference


@pytest.mark.parametrize("name", ["j2d5pt", "j2d9pt-gol", "j2d9pt", "j2d25pt", "j2d13pt",
                                  "j2ds25pt", "j3d7pt", "j3d13pt", "j3d17pt", "j3d27pt",
                                  "poisson", "j1d3pt"])
def test_fp32_within_tolerance(name):
    """fp32 kernels (ebisu_run_host_f32) against the fp64 oracle: relative
    error <= 1e-5 of max |ref| on ragged grids at every fp32 depth, the fast
    path (last extent a multiple of 4) and the naive fallback (odd extent)."""
    st = _shape(name)
    r = st.radius
    rng = eb.SplitMix64(0xF32 + len(name))
    # depths with an fp32 kernel at or below them (gen_instances.F32_2D/3D)
    depths = {"j2d5pt": (4, 8, 12, 16), "j3d7pt": (2, 3, 4)}.get(
        name, (1,) if st.dims == 1 else ((2, 3) if st.dims == 2 and r < 6 else (1, 2)))
    for t in depths:
        if st.dims == 1:
            ext = (301,)
        elif st.dims == 2:
            ext = (2 * r + 1 + rng.randint(0, 300), 4 * (r + 1 + rng.randint(0, 300) // 4))
        else:
            ext = (2 * r + 1 + rng.randint(0, 40), 2 * r + 1 + rng.randint(0, 60),
                   4 * (r + 1 + rng.randint(0, 60) // 4))
        steps = rng.randint(t, 3 * t + 2)
        g = eb.random_grid(ext, rng.next_u64())
        ref = oracle_run(g.cells, taps_of(st), steps)
        out, tr = eb.sweep(g, st, steps, t=t, trace=True, dtype=np.float32)
        if st.dims >= 2:
            assert tr["kernel"] in ("stream2d_tb", "stream3d_tb"), (name, t, tr["kernel"])
        err = np.max(np.abs(out.cells - ref))
        assert err <= FP32_RTOL * np.max(np.abs(ref)), (name, t, ext, steps, err)
    # odd last extent: the fp32 naive kernel
    ext = (2 * r + 9,) * (st.dims - 1) + (2 * r + 7,)
    g = eb.random_grid(ext, 3)
    out, tr = eb.sweep(g, st, 5, trace=True, dtype=np.float32)
    ref = oracle_run(g.cells, taps_of(st), 5)
    assert np.max(np.abs(out.cells - ref)) <= FP32_RTOL * np.max(np.abs(ref))


def test_fp32_full_size_against_fp64_gpu():
    """BASELINE config 2 geometry in fp32 (8192^2, 100 steps) against the fp64
    GPU sweep, which is bitwise equal to the oracle (test_full_size_8192)."""
    from paper_2305_07390_b200 import device

    torch = _torch()
    st = eb.make_benchmark("j2d5pt")
    d64 = device.random_grid_device((8192, 8192), seed=1)
    ref = device.sweep_device(d64, st, 100)
    d32 = d64.float()
    out, tr = device.sweep_device(d32, st, 100, trace=True)
    assert out.dtype == torch.float32 and tr["kernel"] == "stream2d_tb"
    err = (out.double() - ref).abs().max().item()
    assert err <= FP32_RTOL * ref.abs().max().item(), err


def test_config5_geometry_1024_cubed_tb_equals_naive():
    """BASELINE config 5 geometry on one GPU (j3d7pt 1024^3, 8 GiB per array,
    64-bit offsets): the temporal-blocking sweep equals the one-launch-per-step
    naive kernel bitwise (both exact), and composes (run(2t) = run(t)∘run(t))."""
    from paper_2305_07390_b200 import device

    torch = _torch()
    st = eb.make_benchmark("j3d7pt")
    d_in = device.random_grid_device((1024, 1024, 1024), seed=9)
    a = device.sweep_device(d_in, st, 8, t=4)
    b = device.sweep_device(d_in, st, 8, scheme=_native.SCHEME_NAIVE)
    cmp = device.compare_device(a, b)
    assert cmp["mismatches"] == 0, cmp
    del b
    half = device.sweep_device(d_in, st, 4, t=4)
    del d_in
    c = device.sweep_device(half, st, 4, t=4)
    cmp = device.compare_device(a, c)
    assert cmp["mismatches"] == 0, cmp
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", list(CASES_2D))
def test_2d_every_registered_variant_bitwise(name):
    """Every registered 2-D kernel variant (e.g. the shifted-window kernels of
    the large-radius stars) on ragged grids, bitwise against the oracle."""
    st = _shape(name)
    for t in CASES_2D[name]:
        steps = 2 * t + 1
        for ext in ((2 * st.radius + 41, 262), (129, 2 * (2 * st.radius + 70))):
            ref = None
            for scheme in (_native.SCHEME_SM_TILING, _native.SCHEME_DEVICE_TILING):
                for g, v, tr, out in _variants(st, t, ext, steps, scheme):
                    if ref is None:
                        ref = oracle_run(g.cells, taps_of(st), steps)
                    assert np.array_equal(out.cells, ref), (name, t, v, scheme, ext, tr)


def test_concurrent_calls_from_threads():
    """The reference promises pure, thread-safe calls: host
    sweeps issued from several Python threads at once all return the oracle's
    answer and leave their inputs untouched."""
    from concurrent.futures import ThreadPoolExecutor

    cases = [("j2d5pt", (200, 260), 9), ("j3d7pt", (30, 40, 66), 6),
             ("j2d9pt", (150, 200), 7), ("j3d27pt", (20, 30, 34), 4)] * 2
    grids = [eb.random_grid(ext, 300 + i) for i, (_, ext, _) in enumerate(cases)]
    before = [g.cells.copy() for g in grids]

    def run(i):
        name, _, steps = cases[i]
        return eb.reference_run(grids[i], _shape(name), steps)

    with ThreadPoolExecutor(max_workers=4) as ex:
        outs = list(ex.map(run, range(len(cases))))
    for i, (name, _, steps) in enumerate(cases):
        assert np.array_equal(grids[i].cells, before[i])
        ref = oracle_run(before[i], taps_of(_shape(name)), steps)
        assert np.array_equal(outs[i].cells, ref), (name, i)


# Tolerance mode (exact = 0) with uniform coefficients: the reassociated
# kernels (ebisu_trace.arith == reassociated), every registered variant per
# depth, both 2-D schemes, within 1e-12 of max |ref| (north star fp64 bar).
TOL_CASES = {"j2ds25pt": [1, 2], "j2d13pt": [1, 2, 3], "j2d25pt": [1, 2, 3],
             "j2d9pt-gol": [1, 2, 3, 4, 6], "j2d9pt": [1, 2, 3],
             "j3d27pt": [1, 2], "poisson": [1, 2], "j3d17pt": [1, 2]}


@pytest.mark.parametrize("name", list(TOL_CASES))
def test_reassociated_kernels_within_tolerance(name):
    st = _shape(name)
    r = st.radius
    exts = (((2 * r + 41, 262), (129, 2 * (2 * r + 70)), (300, 999)) if st.dims == 2
            else ((37, 71, 134), (2 * r + 3, 300, 66)))
    schemes = ((_native.SCHEME_SM_TILING, _native.SCHEME_DEVICE_TILING) if st.dims == 2
               else (_native.SCHEME_AUTO,))
    seen_ra = 0
    for t in TOL_CASES[name]:
        for ext in exts:
            g = eb.random_grid(ext, 53 + t)
            steps = 3 * t + 1
            ref = oracle_run(g.cells, taps_of(st), steps)
            for scheme in schemes:
                for v in range(16):
                    prm = _native.make_params(t=t, variant=v, scheme=scheme, exact=False)
                    try:
                        out, tr = eb.sweep(g, st, steps, params=prm, trace=True)
                    except Exception as e:  # past the last registered variant
                        assert "variant" in str(e), e
                        break
                    err = np.max(np.abs(out.cells - ref))
                    assert err <= FMA_RTOL * np.max(np.abs(ref)), (name, t, v, scheme, ext, err)
                    seen_ra += tr["arith"] == "reassociated"
    assert seen_ra > 0, name


@pytest.mark.parametrize("name,ext,steps", [("j3d27pt", (512, 512, 512), 500),
                                            ("j2ds25pt", (8192, 8192), 96),
                                            ("j2d13pt", (8192, 8192), 96)])
def test_reassociated_full_size_against_bitwise_gpu(name, ext, steps):
    """BASELINE configs 3/4 at full size and step count: the tolerance-mode
    sweep within 1e-12 of the bitwise sweep (itself pinned to the oracle by
    test_fullsize_parity's golden digests)."""
    from paper_2305_07390_b200 import device

    torch = _torch()
    st = _shape(name)
    d = device.random_grid_device(ext, seed=1)
    a, b, s = torch.empty_like(d), torch.empty_like(d), torch.empty_like(d)
    _, tr = device.sweep_device(d, st, steps, out=a, scratch=s, trace=True,
                                params=_native.make_params(exact=False))
    assert tr["arith"] == "reassociated", tr
    device.sweep_device(d, st, steps, out=b, scratch=s, params=_native.make_params(exact=True))
    cmp = device.compare_device(a, b)
    assert cmp["max_abs_diff"] <= FMA_RTOL * cmp["max_abs_ref"], cmp
    del a, b, s, d
    torch.cuda.empty_cache()


# ---- device tiles of several CTAs (cluster halo exchange, k_halo2d CLU) ------

@pytest.mark.parametrize("name,t", [("j2d5pt", 4), ("j2d5pt", 8), ("j2d9pt-gol", 2),
                                    ("j2d9pt", 2), ("j2d25pt", 2), ("j2d13pt", 2),
                                    ("j2d13pt", 3), ("j2ds25pt", 1), ("j2ds25pt", 2)])
def test_device_tiles_of_cluster_ctas_bitwise(name, t):
    """run_device_tiling with device_tile_grid = (1, CL): CL CTA strips per
    device tile exchange their seam edges through DSMEM every level
    (engine/device.py:145-211's per-step halo exchange); bitwise equal to the
    oracle for widths below, at and above one tile, ragged strips included."""
    st = _shape(name)
    r = st.radius
    rng = eb.SplitMix64(0xC1 + 7 * t + len(name))
    for cl in ((2, 3, 4, 8) if t == 4 else (2, 4, 8)):
        for n1 in (2 * r + 2, 1024 * cl - 64, 1024 * cl, 2 * 1024 * cl + 4 * r + 38):
            n0 = 2 * r + 1 + rng.randint(0, 200)
            steps = t * rng.randint(1, 2)  # whole epochs: every stage is a halo stage
            g = eb.random_grid((n0, n1), rng.next_u64())
            ref = oracle_run(g.cells, taps_of(st), steps)
            prm = _native.make_params(scheme=_native.SCHEME_DEVICE_TILING, t=t,
                                      device_tile_grid=(1, cl))
            out, tr = eb.sweep(g, st, steps, params=prm, trace=True)
            assert tr["kernel"] == "halo2d_tb" and tr["cluster_ctas"] == cl, (cl, tr)
            assert np.array_equal(out.cells, ref), (name, t, cl, (n0, n1), steps)


def test_device_tiles_auto_cluster_full_width():
    """AUTO device tiles on the config-3 geometry pick a cluster when it covers
    the width with fewer computed columns; result bitwise equal to the
    single-CTA tiles (which match the oracle, test_gpu_parity golden cases)."""
    from paper_2305_07390_b200 import device

    torch = _torch()
    st = _shape("j2d13pt")
    d_in = device.random_grid_device((1024, 8192), seed=2)
    one = device.sweep_device(d_in, st, 6, params=_native.make_params(
        scheme=_native.SCHEME_DEVICE_TILING, t=2, device_tile_grid=(1, 1)))
    out, tr = device.sweep_device(d_in, st, 6, scheme=_native.SCHEME_DEVICE_TILING, t=2,
                                  trace=True)
    assert tr["kernel"] == "halo2d_tb"
    assert torch.equal(out, one), tr


def test_host_entry_pageable_and_pinned_buffers_agree():
    """ebisu_run_host stages pageable (numpy) buffers through its pinned slot
    ring with host threads: multi-chunk sizes that are not a multiple of the
    slot size (8-16 MiB), fresh (unfaulted) outputs, aliasing in == out on the host,
    and pinned buffers (direct DMA) all give the same bitwise result."""
    import ctypes

    torch = _torch()
    st = _shape("j2d5pt")
    lib = _native.load()
    sa = _native.StencilArgs(st)
    for ext in ((3001, 1003), (64, 2 * (1 << 21) + 2)):  # 24 MiB, 2 x 16 MiB + 16 B
        g = eb.random_grid(ext, 21)
        ref = eb.sweep(g, st, 9, t=4).cells  # pageable in, fresh pageable out
        src = np.ascontiguousarray(g.cells)
        pin_in = torch.from_numpy(src).pin_memory()
        pin_out = torch.empty_like(pin_in).pin_memory()
        prm = _native.make_params(t=4)
        rc = lib.ebisu_run_host(ctypes.byref(sa.c), 2, _native.extents_c(ext),
                                pin_in.data_ptr(), pin_out.data_ptr(), 9, ctypes.byref(prm), None)
        assert rc == 0, _native.last_error()
        assert np.array_equal(pin_out.numpy(), ref), ext
        inplace = src.copy()  # in == out on the host (allowed by the ABI)
        rc = lib.ebisu_run_host(ctypes.byref(sa.c), 2, _native.extents_c(ext),
                                inplace.ctypes.data, inplace.ctypes.data, 9, ctypes.byref(prm), None)
        assert rc == 0, _native.last_error()
        assert np.array_equal(inplace, ref), ext
        if ext[0] > 100:  # (the oracle on the 2^28-cell case would take minutes)
            assert np.array_equal(ref, oracle_run(g.cells, taps_of(st), 9))
        # the pinned slot ring is released and re-created on demand
        assert lib.ebisu_release_scratch() == 0
        assert np.array_equal(eb.sweep(g, st, 9, t=4).cells, ref), ext


def test_reserve_sms_shrinks_the_persistent_grid():
    """ebisu_params.reserve_sms (the multi-GPU interior call keeps SMs free
    for the concurrent NCCL kernels): fewer resident CTAs, same bits."""
    from paper_2305_07390_b200 import device

    torch = _torch()
    for name, ext in (("j2d5pt", (2048, 2048)), ("j3d7pt", (128, 512, 512))):
        st = _shape(name)
        d_in = device.random_grid_device(ext, seed=8)
        full, tr0 = device.sweep_device(d_in, st, 8, params=_native.make_params(t=4), trace=True)
        part, tr1 = device.sweep_device(d_in, st, 8, params=_native.make_params(
            t=4, reserve_sms=20), trace=True)
        assert torch.equal(full, part), name
        assert tr1["grid_ctas"] < tr0["grid_ctas"], (name, tr0["grid_ctas"], tr1["grid_ctas"])


def test_stream3d_step_kernel_random_user_stencils_bitwise():
    """3-D tap sets without a temporal-blocking kernel run the one-step
    streaming kernel (plane ring in shared memory, k_generic_s3d): random
    user stencils (radius 1-3, random order and coefficients) on ragged and
    odd grids, exact bitwise, FMA within 1e-12, fp32 within 1e-5; the naive
    scheme still runs the naive kernel."""
    rng = eb.SplitMix64(0x53D)
    for case in range(6):
        rad = 1 + rng.randint(0, 2)
        st = _random_shape(rng, 3, rad)
        ext = tuple(2 * rad + 1 + rng.randint(0, 60) for _ in range(2)) + (
            2 * rad + 1 + rng.randint(0, 300),)
        g = eb.random_grid(ext, rng.next_u64())
        steps = rng.randint(1, 5)
        ref = oracle_run(g.cells, taps_of(st), steps)
        out, tr = eb.sweep(g, st, steps, trace=True)
        assert tr["kernel"] == "stream3d_step", tr
        assert np.array_equal(out.cells, ref), (case, ext, steps, st.taps)
        out = eb.sweep(g, st, steps, exact=False)
        assert np.max(np.abs(out.cells - ref)) <= FMA_RTOL * np.max(np.abs(ref))
        out = eb.sweep(g, st, steps, dtype=np.float32)
        assert np.max(np.abs(out.cells - ref)) <= 1e-5 * np.max(np.abs(ref))
        out, tr = eb.sweep(g, st, steps, scheme=_native.SCHEME_NAIVE, trace=True)
        assert tr["kernel"] == "naive_step" and np.array_equal(out.cells, ref)


def test_3d_device_tiles_of_two_ctas_bitwise():
    """run_device_tiling in 3-D with device_tile_grid = (2, 1): the 2-CTA
    cluster tile (seam rows exchanged through DSMEM every level) where one is
    instantiated (j3d7pt t = 2, 3), bitwise equal to the oracle; otherwise the
    one-CTA tile (same result)."""
    st = _shape("j3d7pt")
    for t, ext in ((2, (40, 70, 66)), (3, (33, 130, 64)), (4, (20, 40, 36))):
        g = eb.random_grid(ext, 31 + t)
        ref = oracle_run(g.cells, taps_of(st), 2 * t)
        prm = _native.make_params(scheme=_native.SCHEME_DEVICE_TILING, t=t,
                                  device_tile_grid=(2, 1))
        out, tr = eb.sweep(g, st, 2 * t, params=prm, trace=True)
        assert tr["kernel"] == "stream3d_tb", tr
        assert tr["cluster_ctas"] == (2 if t in (2, 3) else 1), tr
        assert np.array_equal(out.cells, ref), (t, ext)
