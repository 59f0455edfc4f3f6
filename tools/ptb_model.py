"""Paper model vs measured -- run in the build
container, which has the reference package (it is NOT used at run time):

    PYTHONPATH=/root/reference/pkg/src python tools/ptb_model.py

Writes
  profiles/b200_hardware.json   B200 HardwareSpec in the reference's config
                                format (hardware.py:101-129, loadable with
                                stencilplan.hardware.get_hardware(path))
  profiles/r01_ptb_model.json   the reference's own model (model.py:89-113,
                                choose_scheme model.py:417) on that spec for
                                every BASELINE config, beside the measured
                                GCells/s of profiles/r01_bench.json
"""

from __future__ import annotations

import json
import os

from stencilplan.hardware import HardwareSpec, hardware_file_dict  # reference package
from stencilplan.model import choose_scheme
from stencilplan.shapes import StencilShape, make_benchmark
from stencilplan.engine.rst import rst_shared_per_cell

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
MHZ = PEAKS.get("sm_max_mhz", 1965.0)
SMS = 148

# Bandwidths/throughputs of one B200 (bytes/s, flop/s).  HBM: the measured copy
# peak; shared memory: 128 B/clk/SM (B300_MICROARCH.md "smem crossbar BW");
# FP64: 64 DFMA/clk/SM measured (tools/dp_microbench.cu), 2 flops each.
B200 = HardwareSpec(
    name="b200",
    gm_bandwidth=PEAKS["hbm_gbs"] * 1e9,
    sm_bandwidth=SMS * 128 * MHZ * 1e6,
    compute_throughput=SMS * 64 * 2 * MHZ * 1e6,
    cell_bytes=8,
    onchip_capacity_per_block=227 * 1024,
    blocks=SMS,
    device_sync_latency=1.5e-6,
    max_threads_per_sm=2048,
    op_latencies={"dfma": 8.0, "gm_access": 577.0, "sm_access": 29.0},
    op_throughputs={"dfma": 64.0, "gm_access": 5.6, "sm_access": 16.0},
)


def star(dims, rad, name):
    offs = [tuple(d if a == 0 else 0 for a in range(dims)) for d in range(-rad, rad + 1)]
    for axis in range(1, dims):
        for d in list(range(-rad, 0)) + list(range(1, rad + 1)):
            offs.append(tuple(d if a == axis else 0 for a in range(dims)))
    n = len(offs)
    sh = StencilShape(name=name, dims=dims, taps=tuple((o, 1.0 / n) for o in offs),
                      flops_per_cell=2 * n, gm_accesses_per_cell=2,
                      sm_accesses_no_rst=n + 1, sm_accesses_with_rst=n + 1,
                      default_domain=(8192, 8192))
    return StencilShape(name=name, dims=dims, taps=sh.taps, flops_per_cell=2 * n,
                        gm_accesses_per_cell=2, sm_accesses_no_rst=n + 1,
                        sm_accesses_with_rst=float(rst_shared_per_cell(sh)),
                        default_domain=(8192, 8192))


def main():
    bench = json.load(open(os.path.join(ROOT, "profiles", "r01_bench.json")))
    cfg = bench.get("configs", {})
    measured = {
        "j2d5pt": (bench["value"], "config 2, 8192^2 x 1000, t=8"),
        "j3d7pt": (cfg.get("config4_j3d7pt_512", {}).get("value"), "config 4, 512^3 x 500"),
        "j3d27pt": (cfg.get("config4_j3d27pt_512", {}).get("value"), "config 4, 512^3 x 500"),
        "j2d13pt": (cfg.get("config3_j2d13pt_8192_overlapped", {}).get("value"),
                    "config 3, 8192^2, overlapped"),
        "j2ds25pt": (cfg.get("config3_j2ds25pt_8192_overlapped", {}).get("value"),
                     "config 3, 8192^2, overlapped"),
    }
    shapes = {
        "j2d5pt": make_benchmark("j2d5pt"), "j3d7pt": make_benchmark("j3d7pt"),
        "j3d27pt": make_benchmark("j3d27pt"), "j2d13pt": star(2, 3, "j2d13pt"),
        "j2ds25pt": star(2, 6, "j2ds25pt"),
    }
    domains = {"j2d5pt": (8192, 8192), "j3d7pt": (512, 512, 512), "j3d27pt": (512, 512, 512),
               "j2d13pt": (8192, 8192), "j2ds25pt": (8192, 8192)}
    rows = []
    for name, st in shapes.items():
        plan = choose_scheme(B200, st, domain=domains[name])
        a_sm = st.sm_accesses_with_rst
        ptb = B200.sm_bandwidth / (a_sm * B200.cell_bytes) / 1e9  # PAPER.md:65-84, t -> inf
        naive = B200.gm_bandwidth / 16 / 1e9
        meas, what = measured[name]
        rows.append({
            "stencil": name, "measured_gcells": meas, "measured_config": what,
            "model_scheme": plan.scheme, "model_t": plan.t, "model_bottleneck": plan.bottleneck,
            "model_p_gcells": round(plan.predicted_p, 1), "model_v": round(plan.predicted_v, 3),
            "model_pp_gcells": round(plan.predicted_pp, 1),
            "ptb_bound_gcells": round(ptb, 1), "a_sm_rst": a_sm,
            "naive_hbm_roofline_gcells": round(naive, 1),
            "measured_over_model_pp": round(meas / plan.predicted_pp, 2) if meas else None,
            "measured_over_ptb": round(meas / ptb, 2) if meas else None,
        })
    with open(os.path.join(ROOT, "profiles", "b200_hardware.json"), "w") as f:
        json.dump(hardware_file_dict(B200), f, indent=1)
    out = {"_how": "PYTHONPATH=/root/reference/pkg/src python tools/ptb_model.py (reference "
                   "model.choose_scheme on profiles/b200_hardware.json)",
           "hardware": hardware_file_dict(B200), "rows": rows}
    with open(os.path.join(ROOT, "profiles", "r01_ptb_model.json"), "w") as f:
        json.dump(out, f, indent=1)
    for r in rows:
        print(r)


if __name__ == "__main__":
    main()
