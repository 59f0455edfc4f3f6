"""The reference's OWN test suite, unmodified, run against the B200 path.

``baseline/_ref/pkg`` is a copy of the reference package (src + tests) made
by ``__graft_entry__.build()`` in the build container (git-ignored; it
travels to the GPU box with the snapshot).  The suite runs in a subprocess
with ``tests/ref_plugin/b200_swap_plugin.py`` loaded first, which routes
``planner._ENGINES`` and ``stencilplan.engine.run_*`` to the B200 engines
(``paper_2305_07390_b200.stencilplan_bridge``):

* every engine test (test_engine_sm.py, test_engine_device.py), the
  acceptance sweeps c08 (4,000 engine runs bitwise against the numpy
  ``reference_run``), c10 (valid proportion, device syncs), c11 (on-chip
  access accounting), c13 (``cmd_simulate`` reports byte-identical), the
  planner / CLI / service ``simulate`` paths -- all against the GPU engines;
* test_grid.py a second time with ``reference_run`` / ``reference_step``
  also swapped, so its brute-force transcriptions (test_grid.py:43-91) and
  purity checks judge the GPU sweep.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF_PKG = os.path.join(ROOT, "baseline", "_ref", "pkg")
PLUGIN_DIR = os.path.join(ROOT, "tests", "ref_plugin")

pytestmark = pytest.mark.gpu


def _run_suite(tmp_path, targets, swap_run: bool):
    if not os.path.isdir(os.path.join(REF_PKG, "tests")):
        pytest.skip("baseline/_ref/pkg missing (run __graft_entry__.build() where "
                    "/root/reference exists)")
    count_file = tmp_path / "calls.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join(
        [os.path.join(REF_PKG, "src"), PLUGIN_DIR, ROOT, env.get("PYTHONPATH", "")])
    env["EBISU_SWAP_REFERENCE_RUN"] = "1" if swap_run else "0"
    env["EBISU_SWAP_COUNT_FILE"] = str(count_file)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
           "-p", "b200_swap_plugin", "--rootdir", REF_PKG, *targets]
    r = subprocess.run(cmd, cwd=REF_PKG, env=env, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    calls = json.loads(count_file.read_text())
    return calls, tail


def test_reference_suite_with_b200_engines(tmp_path):
    calls, tail = _run_suite(tmp_path, ["tests"], swap_run=False)
    # c08 alone makes 4,000 engine calls
    assert calls["engine"] > 4000, (calls, tail)
    assert " passed" in tail and "failed" not in tail


def test_reference_grid_tests_with_b200_reference_run(tmp_path):
    calls, tail = _run_suite(tmp_path, ["tests/test_grid.py"], swap_run=True)
    assert calls["reference_run"] > 10, (calls, tail)


STUB_SCRIPT = r'''
import importlib.util, json, os, sys
import numpy as np
spec = importlib.util.spec_from_file_location("stencilplan_b200", sys.argv[1])
b200 = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b200)
import stencilplan
from stencilplan import make_benchmark, random_grid, reference_run
from stencilplan.engine import DEVICE_TILING, SM_TILING, ParamError, TilingParams
from stencilplan import planner
from stencilplan.hardware import A100
runs = 0
for name, dom, params in [
        ("j2d5pt", (96, 1024), TilingParams(scheme=SM_TILING, t=7, tile=(256,))),
        ("j3d7pt", (30, 40, 44), TilingParams(scheme=SM_TILING, t=3, tile=(16, 16))),
        ("j2d9pt", (60, 70), TilingParams(scheme=DEVICE_TILING, t=2, tile=(30, 35),
                                          device_tile_grid=(2, 2)))]:
    st = make_benchmark(name)
    g = random_grid(dom, seed=7)
    for steps in (None, 11):
        out, tr = b200.run_b200(g, st, params, steps=steps)
        ref = reference_run(g, st, params.t if steps is None else steps)
        assert np.array_equal(out.cells, ref.cells), (name, steps)
        assert tr.cells_valid > 0 and tr.cells_computed >= tr.cells_valid
        runs += 1
try:
    b200.run_b200(random_grid((12, 20), seed=0), make_benchmark("j2d5pt"),
                  TilingParams(scheme=SM_TILING, t=5, tile=(10,)))
    raise SystemExit("ParamError not raised")
except ParamError as e:
    assert "valid core" in str(e), e
planner._ENGINES = {SM_TILING: b200.run_b200, DEVICE_TILING: b200.run_b200}
suite = planner.SuiteConfig(stencils=["j2d5pt", "j3d7pt", "j3d27pt"],
                            domains={"j2d5pt": [64, 300], "j3d7pt": [20, 40, 40],
                                     "j3d27pt": [16, 30, 30]}, workers=1, seed=77)
payload = planner.cmd_simulate(suite, A100)
assert payload["ok"], payload
print(json.dumps({"runs": runs, "simulated": len(payload["runs"])}))
'''


def test_integration_binding_on_the_reference(tmp_path):
    """INTEGRATION.md §2's binding (tools/stencilplan_b200_engine.py, verbatim)
    on an unmodified copy of the reference: bitwise vs the numpy reference_run,
    ParamError on a bad tile, and cmd_simulate through planner._ENGINES."""
    if not os.path.isdir(os.path.join(REF_PKG, "src")):
        pytest.skip("baseline/_ref/pkg missing")
    from paper_2305_07390_b200 import _native

    script = tmp_path / "stub_check.py"
    script.write_text(STUB_SCRIPT)
    env = dict(os.environ)
    env["PYTHONPATH"] = os.path.join(REF_PKG, "src")
    env["EBISU_LIB"] = _native.LIB_PATH
    r = subprocess.run([sys.executable, str(script),
                        os.path.join(ROOT, "tools", "stencilplan_b200_engine.py")],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["runs"] == 6 and res["simulated"] == 3


def test_cli_simulate_with_b200_engines(tmp_path):
    """the reference CLI's ``simulate`` on the GPU engines
    (``python -m paper_2305_07390_b200.stencilplan_bridge simulate``): every
    suite run goes through planner._simulate_one -> the B200 engine, is
    checked against the reference's numpy oracle (exit code 0 = all bitwise),
    and the report lands where the reference writes it."""
    if not os.path.isdir(os.path.join(REF_PKG, "src")):
        pytest.skip("baseline/_ref/pkg missing")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REF_PKG, "src"), ROOT,
                                         env.get("PYTHONPATH", "")])
    suite = tmp_path / "suite.json"
    suite.write_text(json.dumps({
        "stencils": ["j2d5pt", "j2d9pt-gol", "j3d7pt", "j3d27pt", "j1d3pt"],
        "domains": {"j2d5pt": [96, 200], "j2d9pt-gol": [64, 130], "j3d7pt": [24, 20, 32],
                    "j3d27pt": [20, 18, 16], "j1d3pt": [5000]}}))
    out = tmp_path / "report"
    cmd = [sys.executable, "-m", "paper_2305_07390_b200.stencilplan_bridge", "simulate",
           "--suite", str(suite), "--out", str(out), "--workers", "1"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    rep = json.loads((out / "report.json").read_text())
    runs = rep["runs"]
    assert rep["ok"] and len(runs) == 5, rep
    assert all(rec["oracle"] == "pass" for rec in runs), runs[:3]
    assert "[b200] engine calls: 5 " in r.stderr, r.stderr[-2000:]  # every run on the GPU

