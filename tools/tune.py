"""Tuning sweep for the 2-D kernel on the GPU box (not part of the bench)."""
import itertools, json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_07390_b200 as eb
from paper_2305_07390_b200 import device, _native

name = sys.argv[1] if len(sys.argv) > 1 else "j2d5pt"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
configs = json.loads(sys.argv[3]) if len(sys.argv) > 3 else [[8, 4, 0]]
st = eb.get_shape(name)
ext = (n,) * st.dims
d_in = device.random_grid_device(ext, seed=1)
out = torch.empty_like(d_in); scr = torch.empty_like(d_in)
res = {}
interior = (n - 2 * st.radius) ** st.dims
for cfg in configs:
    t, c, seg = cfg[:3]
    var = cfg[3] if len(cfg) > 3 else 0
    scheme = cfg[4] if len(cfg) > 4 else 0  # 2 sm-tiling (overlapped), 3 device-tiling (halo)
    nt = t * max(1, (240 if st.dims == 2 else 48) // t)
    prm = _native.make_params(scheme=scheme, t=t, lane_cells=c, seg_rows=seg, variant=var,
                              exact=os.environ.get("EBISU_EXACT", "1") == "1")
    try:
        device.sweep_device(d_in, st, nt, out=out, scratch=scr, params=prm)
        torch.cuda.synchronize()
        best = 0
        for _ in range(3):
            _, tr = device.sweep_device(d_in, st, nt, out=out, scratch=scr, params=prm, trace=True)
            best = max(best, interior * nt / (tr["elapsed_ms"] / 1e3) / 1e9)
        res[f"t{t}_c{c}_s{seg}_v{var}_k{scheme}"] = round(best, 1)
        print(f"{name} t={t} C={c} seg={seg} v={var} scheme={scheme}: {best:.1f} GCells/s (grid {tr['grid_ctas']}x{tr['warps_per_cta']}, {tr['kernel']})", flush=True)
    except Exception as e:
        print(f"{name} t={t} C={c} seg={seg} v={var}: ERROR {e}", flush=True)
print(json.dumps(res))
