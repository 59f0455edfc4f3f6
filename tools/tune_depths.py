"""Planner default depths: GCells/s of every catalog shape at every fused depth
1..8 (exact and tolerance mode), AUTO scheme, BASELINE-size grids
(2-D 8192^2, 3-D 512^3), 3 timed sweeps each (best).  The planner's
default_depth / default_depth_tol tables come from this run."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_07390_b200 as eb
from paper_2305_07390_b200 import _native, device
names = sys.argv[1:] or ["j2d5pt", "j2d9pt-gol", "j2d9pt", "j2d25pt", "j2d13pt", "j2ds25pt",
                         "j3d7pt", "j3d13pt", "j3d17pt", "j3d27pt", "poisson"]
grids = {}
for name in names:
    st = eb.get_shape(name)
    n = 8192 if st.dims == 2 else 512
    if st.dims not in grids:
        d = device.random_grid_device((n,) * st.dims, seed=1)
        grids[st.dims] = (d, torch.empty_like(d), torch.empty_like(d))
    d, o, s = grids[st.dims]
    inner = (n - 2 * st.radius) ** st.dims
    res = {}
    for exact in (True, False):
        for t in range(1, 9):
            steps = 240 if st.dims == 2 else 96
            steps = t * max(1, steps // t)
            prm = _native.make_params(t=t, exact=exact)
            try:
                device.sweep_device(d, st, steps, out=o, scratch=s, params=prm)
                best = None
                for _ in range(3):
                    _, tr = device.sweep_device(d, st, steps, out=o, scratch=s, params=prm, trace=True)
                    best = tr if best is None or tr["elapsed_ms"] < best["elapsed_ms"] else best
                if best["t_used"] != t:
                    continue  # composed from a shallower kernel
                res[f"{'x' if exact else 'tol'}{t}"] = (round(inner * steps / best["elapsed_ms"] * 1e3 / 1e9, 1), best["arith"][:3])
            except Exception as exc:
                res[f"{'x' if exact else 'tol'}{t}"] = repr(exc)[:40]
        _, tr = device.sweep_device(d, st, 240 if st.dims == 2 else 96, out=o, scratch=s, exact=exact, trace=True)
        res[f"default_{'x' if exact else 'tol'}"] = (tr["t_used"], round(inner * (240 if st.dims == 2 else 96) / tr["elapsed_ms"] * 1e3 / 1e9, 1))
    print(name, json.dumps(res), flush=True)
