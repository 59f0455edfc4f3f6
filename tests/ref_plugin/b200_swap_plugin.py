"""pytest plugin: run the UNMODIFIED reference test suite against the B200 path.

Loaded with ``-p b200_swap_plugin`` before the reference's conftest imports
``stencilplan.engine`` (tests/test_reference_suite.py drives it), so every
``run_sm_tiling`` / ``run_device_tiling`` / ``planner._ENGINES`` the
reference tests reach is the B200 engine (``stencilplan_bridge.install``).
``EBISU_SWAP_REFERENCE_RUN=1`` also swaps ``stencilplan.reference_run`` /
``reference_step`` (for test_grid.py, whose brute-force transcriptions then
check the GPU sweep).  At session end the number of B200 calls is written to
``$EBISU_SWAP_COUNT_FILE`` so the driver can prove the swap was live.
"""

from __future__ import annotations

import json
import os

import stencilplan

from paper_2305_07390_b200 import stencilplan_bridge

_CALLS = {"engine": 0, "reference_run": 0}


def _counting(fn, key):
    def wrapped(*a, **k):
        _CALLS[key] += 1
        return fn(*a, **k)

    wrapped.__name__ = getattr(fn, "__name__", key)
    return wrapped


_swap_run = os.environ.get("EBISU_SWAP_REFERENCE_RUN") == "1"
stencilplan_bridge.install(stencilplan, engines=True, reference_run=_swap_run)
for _mod, _name in ((stencilplan.engine, "run_sm_tiling"), (stencilplan.engine, "run_device_tiling"),
                    (stencilplan.engine.sm, "run_sm_tiling"),
                    (stencilplan.engine.device, "run_device_tiling")):
    setattr(_mod, _name, _counting(getattr(_mod, _name), "engine"))
stencilplan.planner._ENGINES = {k: _counting(v, "engine")
                                for k, v in stencilplan.planner._ENGINES.items()}
if _swap_run:
    for _mod in (stencilplan, stencilplan.grid):
        _mod.reference_run = _counting(_mod.reference_run, "reference_run")
        _mod.reference_step = _counting(_mod.reference_step, "reference_run")


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("EBISU_SWAP_COUNT_FILE")
    if path:
        with open(path, "w") as f:
            json.dump(dict(_CALLS), f)
