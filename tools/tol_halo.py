import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_07390_b200 as eb
from paper_2305_07390_b200 import _native, device
d = device.random_grid_device((8192, 8192), seed=1); o = torch.empty_like(d); s = torch.empty_like(d)
for name in ("j2ds25pt", "j2d13pt", "j2d25pt", "j2d9pt"):
    st = eb.get_shape(name)
    inner = (8192 - 2 * st.radius) ** 2 * 96
    for scheme in (_native.SCHEME_SM_TILING, _native.SCHEME_DEVICE_TILING):
        for t in (1, 2, 3, 4):
            for exact in (True, False):
                prm = _native.make_params(scheme=scheme, t=t, exact=exact)
                try:
                    device.sweep_device(d, st, 96, out=o, scratch=s, params=prm)
                    _, tr = device.sweep_device(d, st, 96, out=o, scratch=s, params=prm, trace=True)
                    print(name, scheme, t, exact, round(inner / tr["elapsed_ms"] * 1e3 / 1e9, 1), tr["kernel"], tr["arith"], tr["t_used"], flush=True)
                except Exception as exc:
                    print(name, scheme, t, exact, repr(exc)[:50])
