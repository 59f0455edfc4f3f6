"""A/B: j3d7pt 512^3 x 500 (t=4) with the package in cwd; prints the trace."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2305_07390_b200 as eb
from paper_2305_07390_b200 import device
st = eb.make_benchmark("j3d7pt")
ext, steps = (512,) * 3, 500
d = device.random_grid_device(ext, seed=1); o = torch.empty_like(d); s = torch.empty_like(d)
device.sweep_device(d, st, steps, out=o, scratch=s)
best = None
for _ in range(3):
    _, tr = device.sweep_device(d, st, steps, out=o, scratch=s, trace=True)
    best = tr if best is None or tr["elapsed_ms"] < best["elapsed_ms"] else best
print(os.getcwd()[-20:], round(510 ** 3 * steps / best["elapsed_ms"] * 1e3 / 1e9, 1),
      {k: best[k] for k in ("gm_loads", "cells_computed", "device_tiles", "kernel_launches", "grid_ctas",
                            "warps_per_cta", "syncs_device", "syncs_block") if k in best}, flush=True)
