"""j3d7pt 512^3 x 500: every registered kernel variant per depth (exact)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_07390_b200 as eb
from paper_2305_07390_b200 import _native, device
name = sys.argv[1] if len(sys.argv) > 1 else "j3d7pt"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 500
st = eb.get_shape(name)
d = device.random_grid_device((n,) * 3, seed=1)
o = torch.empty_like(d); s = torch.empty_like(d)
for t in (2, 3, 4):
    for v in range(4):
        prm = _native.make_params(t=t, variant=v)
        try:
            device.sweep_device(d, st, steps, out=o, scratch=s, params=prm)
            best = None
            for _ in range(3):
                _, tr = device.sweep_device(d, st, steps, out=o, scratch=s, params=prm, trace=True)
                best = tr if best is None or tr["elapsed_ms"] < best["elapsed_ms"] else best
            g = (n - 2) ** 3 * steps / (best["elapsed_ms"] / 1e3) / 1e9
            print(name, t, v, round(g, 1), best["warps_per_cta"], best["grid_ctas"],
                  round(best["cells_valid"] / best["cells_computed"], 3), flush=True)
        except Exception as exc:
            print(name, t, v, "n/a", repr(exc)[:60])
            break
