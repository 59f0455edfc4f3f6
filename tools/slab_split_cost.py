"""Cost of the multi-GPU epoch split on ONE GPU (no exchange): a middle rank's
slab (8192 owned rows + 2 x t*R ghost rows, 8192 columns, j2d5pt, t=8) swept
for 1000 steps as the slab driver does it -- per epoch two band calls and one
interior call (reserve_sms=2), each ranged -- vs one plain sweep of the same
slab.  Bounds the per-rank efficiency the overlapped driver can reach."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_07390_b200 as eb
from paper_2305_07390_b200 import device
from paper_2305_07390_b200.distributed import _default_step, INTERIOR_RESERVE_SMS

st = eb.make_benchmark("j2d5pt")
t, H, n, steps = 8, 8, 8192, 1000
rows = n + 2 * H
a = device.random_grid_device((rows, n), seed=1)
b = torch.empty_like(a)
s = torch.empty_like(a)
step = _default_step(st, True)
lo, hi, inner = (H, 2 * H), (rows - 2 * H, rows - H), (2 * H, rows - 2 * H)
comm = torch.cuda.Stream()
cur = torch.cuda.current_stream()

def split_sweep(reserve):
    src, dst = a, b
    for e in range(steps // t):
        comm.wait_stream(cur)
        with torch.cuda.stream(comm):
            step(src, dst, None, t, t, planes=lo, frame_ready=e > 0)
            step(src, dst, None, t, t, planes=hi, frame_ready=e > 0)
        step(src, dst, None, t, t, planes=inner, frame_ready=e > 0, reserve_sms=reserve)
        cur.wait_stream(comm)
        src, dst = dst, src
    return

def timed(f):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); f(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3

full_ms, _ = timed(lambda: device.sweep_device(a, st, steps, out=b, scratch=s, t=t))
split0_ms, host0 = timed(lambda: split_sweep(0))
split2_ms, host2 = timed(lambda: split_sweep(INTERIOR_RESERVE_SMS))
cells = (n - 2) * (rows - 2) * steps
print(f"full sweep {full_ms:.2f} ms ({cells / full_ms / 1e6:.0f} GCells/s); "
      f"split reserve 0: {split0_ms:.2f} ms (host {host0:.1f} ms), "
      f"split reserve {INTERIOR_RESERVE_SMS}: {split2_ms:.2f} ms (host {host2:.1f} ms); "
      f"efficiency bound {full_ms / split2_ms:.3f}")

# Deep halos (SlabSweep exchange_every=K): a middle rank sweeps its slab plus
# K*t*R ghost planes per face in ONE persistent call per K epochs; the
# exchange would sit between calls.  Efficiency bound vs the plain sweep of
# the owned rows alone.
own = torch.empty((n, n), dtype=torch.float64, device="cuda")
own.copy_(a[H:H + n])
o2 = torch.empty_like(own); s2 = torch.empty_like(own)
base_ms, _ = timed(lambda: device.sweep_device(own, st, steps, out=o2, scratch=s2, t=t))
for K in (4, 8, 16):
    G = K * t
    slab = device.random_grid_device((n + 2 * G, n), seed=2)
    sb = torch.empty_like(slab); ss = torch.empty_like(slab)

    def deep():
        src, dst = slab, sb
        done = 0
        while done < steps:
            d = min(K * t, steps - done)
            device.sweep_device(src, st, d, out=dst, scratch=ss, t=t)
            src, dst = dst, src
            done += d

    ms, host = timed(deep)
    print(f"deep halo K={K} (ghost {G} planes/face): {ms:.2f} ms vs owned-only sweep "
          f"{base_ms:.2f} ms -> efficiency bound {base_ms / ms:.3f}")
