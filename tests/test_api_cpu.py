"""Host-side API behaviour that needs no GPU: shapes, grids, validation and
error messages (the reference's test_grid.py / test_engine_*.py error cases),
and the no-fallback rule."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2305_07390_b200 as eb
from paper_2305_07390_b200 import _native
from paper_2305_07390_b200.engine import (
    SM_TILING,
    DEVICE_TILING,
    ParamError,
    TilingParams,
    onchip_charges,
    rst_shared_per_cell,
)
from paper_2305_07390_b200.grid import Grid


def test_catalog_and_errors():
    assert len(eb.BENCHMARK_NAMES) == 10
    with pytest.raises(eb.CatalogError):
        eb.make_benchmark("nope")
    with pytest.raises(ValueError, match="expected 5 coefficients"):
        eb.make_benchmark("j2d5pt", coefficients=[1.0])
    s = eb.make_benchmark("j3d27pt")
    assert s.radius == 1 and len(s.taps) == 27 and s.dims == 3
    assert eb.get_shape("j2ds25pt").radius == 6 and len(eb.get_shape("j2ds25pt").taps) == 25
    assert eb.get_shape("j2d13pt").radius == 3 and len(eb.get_shape("j2d13pt").taps) == 13


def test_shape_invariants():
    with pytest.raises(ValueError, match="zero offset"):
        eb.StencilShape("x", 1, (((1,), 1.0),), 2, 2, 2, 1.0)
    with pytest.raises(ValueError, match="duplicate"):
        eb.StencilShape("x", 1, (((0,), 1.0), ((0,), 1.0)), 2, 2, 3, 1.0)
    with pytest.raises(ValueError, match="taps\\+1"):
        eb.StencilShape("x", 1, (((0,), 1.0),), 2, 2, 5, 1.0)


def test_rst_charges_match_catalog():
    # engine/rst.py reproduces the catalog "w/ RST" column (test_engine_sm.py:157-165)
    for name in eb.BENCHMARK_NAMES:
        st = eb.make_benchmark(name)
        assert float(rst_shared_per_cell(st)) == st.sm_accesses_with_rst, name
    sh, rg = onchip_charges(eb.make_benchmark("j3d7pt"), True)
    assert sh + rg == 8 and float(sh) == 4.5


def test_grid_validation_messages():
    st = eb.make_benchmark("j2d5pt")
    with pytest.raises(ValueError, match="2-D"):
        eb.reference_step(eb.random_grid((10,), seed=0), st)
    with pytest.raises(ValueError, match="too small"):
        eb.reference_step(eb.random_grid((4, 10), seed=0), eb.make_benchmark("j2d9pt"))
    with pytest.raises(ValueError, match="boundary"):
        Grid(np.zeros((4, 4)), "wrap")
    with pytest.raises(ValueError, match=">= 0"):
        eb.reference_run(eb.random_grid((9, 9), seed=0), st, -1)


def test_zero_steps_is_identity_copy():
    st = eb.make_benchmark("j2d9pt")
    g = eb.random_grid((12, 12), seed=1)
    out = eb.reference_run(g, st, 0)
    assert np.array_equal(out.cells, g.cells)
    assert out.cells is not g.cells


def test_tiling_params_errors():
    with pytest.raises(ParamError, match="scheme"):
        TilingParams(scheme="bogus", t=1, tile=(8,))
    with pytest.raises(ParamError, match="depth"):
        TilingParams(scheme=SM_TILING, t=0, tile=(8,))
    st = eb.make_benchmark("j2d5pt")
    g = eb.random_grid((12, 20), seed=0)
    with pytest.raises(ParamError, match="valid core"):
        eb.run_sm_tiling(g, st, TilingParams(scheme=SM_TILING, t=5, tile=(10,)))
    with pytest.raises(ParamError, match="scheme"):
        eb.run_sm_tiling(g, st, TilingParams(scheme=DEVICE_TILING, t=1, tile=(10, 10)))
    with pytest.raises(ParamError):
        eb.run_device_tiling(eb.random_grid((16, 16), seed=0), st,
                             TilingParams(scheme=DEVICE_TILING, t=6, tile=(3, 3),
                                          device_tile_grid=(2, 2)))
    with pytest.raises(ParamError, match="tile extents"):
        eb.run_sm_tiling(g, st, TilingParams(scheme=SM_TILING, t=1, tile=(10, 10)))


def test_random_grid_matches_reference_digest(golden):
    from conftest import sha256

    for rec in golden["cases"][:6]:
        g = eb.random_grid(rec["extents"], rec["seed"])
        assert sha256(g.cells) == rec["input_sha256"]


def test_no_cpu_fallback_without_gpu(monkeypatch):
    # With no device (this container) or no library, the product raises --
    # it never computes the sweep on the host.
    st = eb.make_benchmark("j2d5pt")
    g = eb.random_grid((16, 16), seed=0)
    try:
        lib_ok = _native.available()
    except Exception:
        lib_ok = False
    if lib_ok and _native.device_count() > 0:
        pytest.skip("a GPU is visible; covered by the gpu tests")
    with pytest.raises((_native.NativeError, _native.NativeUnavailable)):
        eb.reference_run(g, st, 3)
    monkeypatch.setattr(_native, "LIB_PATH", "/nonexistent/libebisu.so")
    monkeypatch.setattr(_native, "_lib", None)
    with pytest.raises(_native.NativeUnavailable):
        eb.reference_run(g, st, 3)


def test_bridge_cli_runs_the_reference_front_end_without_gpu(tmp_path):
    """`python -m paper_2305_07390_b200.stencilplan_bridge` hands argv to the
    unmodified reference CLI after swapping its engines (no GPU work for
    `catalog`): the wiring the GPU test's `simulate` run relies on."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    src = None
    for cand in (os.path.join(ROOT, "baseline", "_ref", "pkg", "src"),
                 "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(cand, "stencilplan")):
            src = cand
            break
    if src is None:
        import pytest

        pytest.skip("reference package not available")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([src, ROOT, env.get("PYTHONPATH", "")])
    r = subprocess.run([sys.executable, "-m", "paper_2305_07390_b200.stencilplan_bridge",
                        "catalog"], cwd=str(tmp_path), env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "j2d5pt" in r.stdout and "j3d27pt" in r.stdout
    assert "[b200] engine calls: 0" in r.stderr
