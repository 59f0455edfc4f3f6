import ctypes, time, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_07390_b200 as eb
from paper_2305_07390_b200 import _native, device
st = eb.make_benchmark("j2d5pt")
g = eb.random_grid((8192, 8192), 1)
lib = _native.load()
sa = _native.StencilArgs(st); ext = _native.extents_c((8192, 8192)); prm = _native.make_params(t=8)
def tm(f, reps=2):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return round((time.perf_counter() - t0) / reps * 1e3, 1)
print("reference_run ms", tm(lambda: eb.reference_run(g, st, 1000)))
src = np.ascontiguousarray(g.cells)
dst = np.empty_like(src); dst[:] = 0
def host(dst_):
    rc = lib.ebisu_run_host(ctypes.byref(sa.c), 2, ext, src.ctypes.data, dst_.ctypes.data, 1000, ctypes.byref(prm), None)
    assert rc == 0
print("run_host prefaulted dst ms", tm(lambda: host(dst)))
print("run_host fresh dst ms", tm(lambda: host(np.empty_like(src))))
d = device.random_grid_device((8192, 8192), 1); o = torch.empty_like(d); s = torch.empty_like(d)
print("device sweep ms", tm(lambda: device.sweep_device(d, st, 1000, out=o, scratch=s)))
print("device sweep no scratch ms", tm(lambda: device.sweep_device(d, st, 1000, out=o)))
