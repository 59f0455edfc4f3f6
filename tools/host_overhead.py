"""Host time per ranged sweep call (the slab driver's per-epoch calls)."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_07390_b200 as eb
from paper_2305_07390_b200 import device, _native
from paper_2305_07390_b200.distributed import _default_step
st = eb.make_benchmark("j2d5pt")
a = device.random_grid_device((8208, 8192), seed=1); b = torch.empty_like(a)
step = _default_step(st, True)
step(a, b, None, 8, 8, planes=(8, 16), frame_ready=False)
torch.cuda.synchronize()
N = 300
for name, planes in (("band", (8, 16)), ("interior", (16, 8192))):
    t0 = time.perf_counter()
    for _ in range(N):
        step(a, b, None, 8, 8, planes=planes, frame_ready=True, reserve_sms=2)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name}: host {1e6 * (t1 - t0) / N:.1f} us/call, total incl. GPU {1e6 * (t2 - t0) / N:.1f} us/call", flush=True)
# raw ctypes call cost without Python wrapper logic
lib = _native.load(); sargs = _native.StencilArgs(st); ext = _native.extents_c((8208, 8192))
prm = _native.make_params(t=8, out_planes=(8, 16), frame_ready=True)
t0 = time.perf_counter()
for _ in range(N):
    lib.ebisu_run_device(ctypes.byref(sargs.c), 2, ext, a.data_ptr(), b.data_ptr(), None, 8, ctypes.byref(prm), device._stream_ptr(), None)
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"raw C call (band): host {1e6 * (t1 - t0) / N:.1f} us/call")
