"""Reference-semantics ExecutionTrace counters (paper_2305_07390_b200.accounting)
against the golden traces of the UNMODIFIED reference engines
(tests/golden/traces.json, made by tests/golden/make_trace_golden.py from
engine/sm.py and engine/device.py).  CPU only: no kernel runs."""

from __future__ import annotations

import hashlib
import json
import os
from fractions import Fraction

import pytest

from conftest import GOLDEN_DIR
from paper_2305_07390_b200 import accounting
from paper_2305_07390_b200.engine import TilingParams
from paper_2305_07390_b200.shapes import make_benchmark


def _cases():
    with open(os.path.join(GOLDEN_DIR, "traces.json")) as f:
        return json.load(f)["cases"]


CASES = _cases()


def _params(p):
    return TilingParams(scheme=p["scheme"], t=p["t"], tile=tuple(p["tile"]),
                        device_tile_grid=tuple(p["device_tile_grid"])
                        if p["device_tile_grid"] else None,
                        lazy=p["lazy"], rst=p["rst"], prefetch=p["prefetch"],
                        transpose_halo=p["transpose_halo"])


def test_fixture_covers_both_schemes_every_shape_and_the_phase_cap():
    assert len(CASES) > 900
    assert {c["params"]["scheme"] for c in CASES} == {"sm-tiling", "device-tiling"}
    assert len({c["stencil"] for c in CASES}) >= 10
    assert max(c["phases_len"] for c in CASES) == accounting.PHASE_CAP + 1


@pytest.mark.parametrize("idx", range(0, len(CASES)))
def test_counters_equal_reference(idx):
    case = CASES[idx]
    st = make_benchmark(case["stencil"])
    params = _params(case["params"])
    c = accounting.reference_counters([o for o, _ in st.taps], st.dims, case["extents"], params)
    for k, v in case["counters"].items():
        assert getattr(c, k) == v, k
    assert c.syncs_block == case["syncs"]["block"]
    assert c.syncs_device == case["syncs"]["device"]
    assert c.onchip_shared == Fraction(*case["onchip_shared"])
    assert c.onchip_register == Fraction(*case["onchip_register"])
    phases = [[t, n] for t, n in c.wall_phases]
    assert len(phases) == case["phases_len"]
    assert phases[:6] == case["phases_head"]
    assert hashlib.sha256(json.dumps(phases).encode()).hexdigest() == case["phases_sha256"]
