"""A/B of 2-D kernels with the package in cwd: fp32 j2d5pt, j2d13pt, j2ds25pt, j2d9pt."""
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2305_07390_b200 as eb
from paper_2305_07390_b200 import device
d64 = device.random_grid_device((8192, 8192), seed=1)
res = {}
for name, dt, steps in (("j2d5pt", "f32", 1000), ("j2d13pt", "f64", 96), ("j2ds25pt", "f64", 96),
                        ("j2d9pt", "f64", 96), ("j2d9pt-gol", "f64", 96), ("j2d25pt", "f64", 96)):
    st = eb.get_shape(name)
    d = d64.float() if dt == "f32" else d64
    o = torch.empty_like(d); s = torch.empty_like(d)
    device.sweep_device(d, st, steps, out=o, scratch=s)
    best = 1e9
    for _ in range(3):
        _, tr = device.sweep_device(d, st, steps, out=o, scratch=s, trace=True)
        best = min(best, tr["elapsed_ms"])
    res[f"{name}_{dt}_t{tr['t_used']}"] = round((8192 - 2 * st.radius) ** 2 * steps / best * 1e3 / 1e9, 1)
print(os.getcwd()[-12:], json.dumps(res), flush=True)
