"""Device tiles of CL CTAs (cluster halo exchange) vs single-CTA tiles:
GCells/s at 8192^2, 96 steps (BASELINE config 3 geometry), exact mode.
python tools/clu_bench.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_07390_b200 as eb  # noqa: E402
from paper_2305_07390_b200 import _native, device  # noqa: E402

d = device.random_grid_device((8192, 8192), seed=1)
o = torch.empty_like(d)
s = torch.empty_like(d)
for name, depths in (("j2d13pt", (2, 3)), ("j2ds25pt", (1, 2)), ("j2d5pt", (4, 8)),
                     ("j2d9pt", (2,)), ("j2d25pt", (2,))):
    st = eb.get_shape(name)
    inner = (8192 - 2 * st.radius) ** 2 * 96
    for t in depths:
        row = {}
        for cl in (0, 1, 2, 4, 8):
            prm = _native.make_params(scheme=_native.SCHEME_DEVICE_TILING, t=t,
                                      device_tile_grid=(1, cl))
            try:
                device.sweep_device(d, st, 96, out=o, scratch=s, params=prm)
                best = None
                for _ in range(2):
                    _, tr = device.sweep_device(d, st, 96, out=o, scratch=s, params=prm, trace=True)
                    if best is None or tr["elapsed_ms"] < best["elapsed_ms"]:
                        best = tr
                row[f"cl{cl}"] = (round(inner / (best["elapsed_ms"] / 1e3) / 1e9, 1),
                                  best["cluster_ctas"], best["grid_ctas"])
            except Exception as exc:
                row[f"cl{cl}"] = repr(exc)[:80]
        prm = _native.make_params(scheme=_native.SCHEME_SM_TILING, t=t)
        _, tr = device.sweep_device(d, st, 96, out=o, scratch=s, params=prm, trace=True)
        row["overlapped"] = round(inner / (tr["elapsed_ms"] / 1e3) / 1e9, 1)
        print(name, t, json.dumps(row), flush=True)
