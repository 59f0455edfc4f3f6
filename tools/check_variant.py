"""Bitwise check + timing of one registered kernel variant (GPU box):
python tools/check_variant.py NAME T VARIANT [EXT ...]  -- compares against the
C oracle on small ragged grids, then times the BASELINE size."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2305_07390_b200 as eb
from oracle import c_oracle
from paper_2305_07390_b200 import _native, device

name, t, var = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
st = eb.get_shape(name)
taps = [(tuple(o), c) for o, c in st.taps]
cases = [(20, 45, 71), (33, 64, 64), (40, 130, 70), (17, 200, 66), (70, 97, 300)]
if st.dims == 2:
    cases = [(45, 71), (200, 257), (64, 1024)]
prm = _native.make_params(t=t, variant=var)
ok = True
for ext in cases:
    g = eb.random_grid(ext, 3)
    for steps in (t, 3 * t + 1):
        out, tr = eb.sweep(g, st, steps, params=prm, trace=True)
        ref = c_oracle.reference_run(g.cells, taps, steps)
        same = np.array_equal(out.cells, ref)
        ok &= same
        if not same:
            bad = np.argwhere(out.cells != ref)
            print("MISMATCH", ext, steps, len(bad), bad[:5].tolist(), flush=True)
print(name, "t", t, "variant", var, "bitwise" if ok else "FAILED", flush=True)
n = int(os.environ.get("N", "512" if st.dims == 3 else "8192"))
steps = int(os.environ.get("STEPS", "500" if st.dims == 3 else "1000"))
d = device.random_grid_device((n,) * st.dims, seed=1)
o, s = torch.empty_like(d), torch.empty_like(d)
device.sweep_device(d, st, steps, out=o, scratch=s, params=prm)
torch.cuda.synchronize()
best = None
for _ in range(3):
    _, tr = device.sweep_device(d, st, steps, out=o, scratch=s, params=prm, trace=True)
    best = tr if best is None or tr["elapsed_ms"] < best["elapsed_ms"] else best
g = (n - 2 * st.radius) ** st.dims * steps / best["elapsed_ms"] / 1e6
print(f"{name} {n}^{st.dims} x{steps} t={t} v={var}: {g:.1f} GCells/s "
      f"grid {best['grid_ctas']}x{best['warps_per_cta']} launches {best['kernel_launches']} "
      f"V={best['cells_valid'] / max(1, best['cells_computed']):.3f}", flush=True)
sys.exit(0 if ok else 1)
