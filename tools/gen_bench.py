"""Resident-tile kernel (any tap set) vs the one-launch-per-step kernel:
GCells/s per depth on the shapes that have no specialised kernel
(j1d3pt, reversed-order catalog stars = user tap sets).
python tools/gen_bench.py [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_07390_b200 as eb  # noqa: E402
from paper_2305_07390_b200 import _native, device  # noqa: E402


def rev(name):
    st = eb.get_shape(name)
    n = len(st.taps)
    return eb.StencilShape(name + "-rev", st.dims, tuple(reversed(st.taps)), 2 * n, 2, n + 1,
                           float(min(4, n + 1)))


def run(st, ext, steps, **kw):
    d = device.random_grid_device(ext, seed=1)
    o = torch.empty_like(d)
    s = torch.empty_like(d)
    device.sweep_device(d, st, steps, out=o, scratch=s, **kw)
    best = None
    for _ in range(2):
        _, tr = device.sweep_device(d, st, steps, out=o, scratch=s, trace=True, **kw)
        if best is None or tr["elapsed_ms"] < best["elapsed_ms"]:
            best = tr
    inner = 1
    for n in ext:
        inner *= n - 2 * st.radius
    return round(inner * steps / (best["elapsed_ms"] / 1e3) / 1e9, 1), best


steps = int(sys.argv[1]) if len(sys.argv) > 1 else 64
res = {}
for st, ext in ((eb.get_shape("j1d3pt"), (8388608 * 4,)), (rev("j2d5pt"), (8192, 8192)),
                (rev("j2d9pt-gol"), (8192, 8192)), (rev("j2d13pt"), (8192, 8192)),
                (rev("j3d7pt"), (512, 512, 512)), (rev("j3d27pt"), (512, 512, 512))):
    r = {}
    g, tr = run(st, ext, steps, scheme=_native.SCHEME_NAIVE)
    r["naive"] = g
    g, tr = run(st, ext, steps)
    r["auto"] = (g, tr["kernel"], tr["t_used"])
    for t in (1, 2, 3, 4, 6, 8, 12, 16):
        try:
            g, tr = run(st, ext, steps, scheme=_native.SCHEME_RESIDENT, t=t)
            r[f"t{t}"] = g
        except Exception as exc:  # no tile fits
            r[f"t{t}"] = repr(exc)[:60]
    res[st.name] = r
    print(st.name, json.dumps(r), flush=True)
