"""One sweep of a reversed-order (user) 3-D stencil: the stream3d_step kernel (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_07390_b200 as eb
from paper_2305_07390_b200 import device
name = sys.argv[1] if len(sys.argv) > 1 else "j3d7pt"
st0 = eb.get_shape(name)
n = len(st0.taps)
st = eb.StencilShape(name + "-rev", 3, tuple(reversed(st0.taps)), 2 * n, 2, n + 1, float(min(4, n + 1)))
d = device.random_grid_device((512, 512, 512), seed=1); o = torch.empty_like(d); s = torch.empty_like(d)
for _ in range(2):
    _, tr = device.sweep_device(d, st, 4, out=o, scratch=s, trace=True)
print(tr)
