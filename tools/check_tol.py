"""Tolerance-mode (exact = 0) check + timing of one stencil on the GPU box:
python tools/check_tol.py NAME T [VARIANT]  -- max|gpu - oracle| / max|oracle|
on small ragged grids (C oracle, reference order), then GCells/s at the
BASELINE size in tolerance and exact mode."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2305_07390_b200 as eb
from oracle import c_oracle
from paper_2305_07390_b200 import _native, device

name, t = sys.argv[1], int(sys.argv[2])
var = int(sys.argv[3]) if len(sys.argv) > 3 else 0
st = eb.get_shape(name)
taps = [(tuple(o), c) for o, c in st.taps]
cases = [(20, 45, 71), (33, 64, 64), (40, 130, 70), (70, 97, 300)]
if st.dims == 2:
    cases = [(45, 71), (200, 257), (64, 1024), (300, 999)]
SCHEME = int(os.environ.get("SCHEME", "0"))  # 2 sm-tiling, 3 device-tiling
prm = _native.make_params(scheme=SCHEME, t=t, variant=var, exact=False)
worst = 0.0
for ext in cases:
    g = eb.random_grid(ext, 3)
    for steps in (t, 3 * t + 1, 40):
        out, tr = eb.sweep(g, st, steps, params=prm, trace=True)
        ref = c_oracle.reference_run(g.cells, taps, steps)
        rel = float(np.max(np.abs(out.cells - ref)) / np.max(np.abs(ref)))
        worst = max(worst, rel)
print(f"{name} t={t} v={var} tolerance mode: max rel err {worst:.3e} "
      f"({'OK' if worst <= 1e-12 else 'FAIL'} vs 1e-12), kernel {tr['kernel']}", flush=True)
n = int(os.environ.get("N", "512" if st.dims == 3 else "8192"))
steps = int(os.environ.get("STEPS", "500" if st.dims == 3 else "96"))
d = device.random_grid_device((n,) * st.dims, seed=1)
o, s = torch.empty_like(d), torch.empty_like(d)
for mode, p in (("tol", prm), ("exact", _native.make_params(scheme=SCHEME, t=t, variant=0, exact=True))):
    try:
        device.sweep_device(d, st, steps, out=o, scratch=s, params=p)
        torch.cuda.synchronize()
        best = None
        for _ in range(3):
            _, tr = device.sweep_device(d, st, steps, out=o, scratch=s, params=p, trace=True)
            best = tr if best is None or tr["elapsed_ms"] < best["elapsed_ms"] else best
        gc = (n - 2 * st.radius) ** st.dims * steps / best["elapsed_ms"] / 1e6
        print(f"  {mode}: {name} {n}^{st.dims} x{steps} t={t}: {gc:.1f} GCells/s "
              f"grid {best['grid_ctas']}x{best['warps_per_cta']} "
              f"V={best['cells_valid'] / max(1, best['cells_computed']):.3f}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"  {mode}: ERROR {e}", flush=True)
sys.exit(0 if worst <= 1e-12 else 1)
