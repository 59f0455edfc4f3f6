"""Single sweep for ncu captures: python tools/prof_run.py NAME N STEPS T [variant]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_07390_b200 as eb
from paper_2305_07390_b200 import device, _native
name, n, steps, t = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
var = int(sys.argv[5]) if len(sys.argv) > 5 else 0
st = eb.get_shape(name)
d_in = device.random_grid_device((n,) * st.dims, seed=1)
out = torch.empty_like(d_in); scr = torch.empty_like(d_in)
scheme = int(sys.argv[6]) if len(sys.argv) > 6 else 0
# EBISU_PERSISTENT=0: one launch per epoch (ncu cannot replay a cooperative
# cluster launch)
# EBISU_EXACT=0: tolerance mode (reassociated kernels for uniform coefficients)
prm = _native.make_params(scheme=scheme, t=t, variant=var,
                          persistent=os.environ.get("EBISU_PERSISTENT", "1") != "0",
                          exact=os.environ.get("EBISU_EXACT", "1") != "0",
                          # EBISU_DTG=n: device tiles of n CTAs (cluster halo exchange)
                          device_tile_grid=(1, int(os.environ.get("EBISU_DTG", "0"))))
for _ in range(2):
    _, tr = device.sweep_device(d_in, st, steps, out=out, scratch=scr, params=prm, trace=True)
print(tr)
