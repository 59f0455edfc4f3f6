#!/usr/bin/env python
"""Benchmark: BASELINE.json metric "GCells/s (fp64)" on the iterated Jacobi sweep.

Workload (N=1, BASELINE config 2): j2d5pt fp64, 8192 x 8192 grid, one bench
step = one full 1000-time-step sweep (reference_run(grid, j2d5pt, 1000)),
synthetic SplitMix64 input (seed 1) generated in HBM, exact (bitwise) mode.
GCells/s counts interior cell updates: (8192-2)^2 x 1000 per step.

Lines printed (rank 0, one JSON line):
  value      device-timed GCells/s over all ranks (CUDA events, max over ranks)
  e2e        same metric through the public C-ABI host call (ebisu_run_host),
             pinned host buffers, H2D + sweep + D2H inside the timed region
  roofline   dominant kernel (stream2d_tb) vs the measured HBM copy peak;
             algorithmic bytes = 16 B per cell-step (the naive sweep's load+store)
  cpu_baseline  the numpy oracle port (1 thread) on a bounded sample
`--impl reference` runs the oracle port (all host threads) instead.

Multi-GPU (torchrun, N>1): slab decomposition along axis 0 with a t*R-deep
halo exchanged over NCCL each epoch (paper_2305_07390_b200.distributed);
per-GPU work is fixed (weak scaling: 8192 x 8192 interior rows per rank).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N0 = N1 = 8192
TSTEPS = 1000
STENCIL = "j2d5pt"
DEPTH = 8
ALG_BYTES_PER_CELL_STEP = 16  # 8 B load + 8 B store of the naive sweep


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm),
                "reasons": sorted(reasons)}


def cpu_oracle_sample(seconds_target: float = 12.0, threads: int = 1) -> dict:
    """Oracle port (numpy restatement of reference_run) on the host."""
    from oracle import reference_run, reference_run_threaded
    from paper_2305_07390_b200.rng import uniform_array
    from paper_2305_07390_b200.shapes import make_benchmark

    st = make_benchmark(STENCIL)
    taps = [(tuple(o), c) for o, c in st.taps]
    cells = uniform_array(1, N0 * N1).reshape(N0, N1)
    run = (lambda c, t: reference_run(c, taps, t)) if threads == 1 else \
        (lambda c, t: reference_run_threaded(c, taps, t, threads))
    run(cells[:256], 1)  # warm
    t0 = time.perf_counter()
    steps = 0
    while True:
        run(cells, 1)
        steps += 1
        if time.perf_counter() - t0 >= seconds_target or steps >= 50:
            break
    dt = time.perf_counter() - t0
    gc = (N0 - 2) * (N1 - 2) * steps / dt / 1e9
    return {"value": gc, "unit": "GCells/s", "cores": threads, "kind": "port",
            "sample": f"{STENCIL} fp64 {N0}x{N1}, {steps} time step(s) of oracle/stencil_oracle."
                      f"reference_run{'_threaded' if threads > 1 else ''} in {dt:.1f} s"}


def lib_sha16() -> str:
    import hashlib

    from paper_2305_07390_b200 import _native

    h = hashlib.sha256()
    with open(_native.LIB_PATH, "rb") as f:
        for chunk in iter(lambda: f.read(1 << 20), b""):
            h.update(chunk)
    return h.hexdigest()[:16]


def measure_dram_traffic(tsteps: int, t: int, timeout: int = 300):
    """DRAM bytes (read + write) of ONE launch of the headline kernel, measured
    in this run: ncu (metrics only, one k_stream2d launch of the same sweep,
    tools/prof_run.py) in a subprocess after the timed region.  Returns
    (bytes or None, provenance dict).  A byte count, not a timing: nothing
    timed here runs under the profiler."""
    src = {"tool": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
                   "(in-run subprocess, one k_stream2d launch)",
           "workload": f"{STENCIL} {N0}x{N1}, {tsteps} steps, t={t}"}
    try:
        src["lib_sha16"] = lib_sha16()
        cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum",
               "--print-units", "base", "--clock-control", "none", "-k", "regex:k_stream2d",
               "-c", "1", "--csv", sys.executable, os.path.join(ROOT, "tools", "prof_run.py"),
               STENCIL, str(N0), str(tsteps), str(t)]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
        import csv
        import io

        rows = list(csv.reader(io.StringIO(r.stdout)))
        start = next(i for i, row in enumerate(rows) if "Metric Name" in row)
        rows = rows[start:]
        hdr = rows[0]
        name_i, val_i = hdr.index("Metric Name"), hdr.index("Metric Value")
        unit_i = hdr.index("Metric Unit")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        tot = 0.0
        seen = set()
        for row in rows[1:]:
            if row[name_i] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                tot += float(row[val_i].replace(",", "")) * scale.get(row[unit_i], 1)
                seen.add(row[name_i])
        if len(seen) != 2:
            raise RuntimeError(f"metrics missing (rc {r.returncode}): {r.stderr[-200:]}")
        return tot, src
    except Exception as exc:  # ncu absent / no permission: report, do not guess
        src["error"] = repr(exc)[:300]
        return None, src


# the paper's PTB bound THR = B_sc / (a_sm * S), a_sm = the
# catalog's per-cell shared accesses with RST (StencilShape.sm_accesses_with_rst,
# shapes.py:128-140), B_sc = 128 B/clk/SM of shared memory
SMEM_B_PER_CLK_PER_SM = 128


def ptb_fraction(stencil: str, gcells: float, sm_mhz, sms: int = 148, elem: int = 8) -> dict:
    """Measured GCells/s vs the paper's PTB bound B_smem / (a_sm * S)
    (SURVEY.md §8d), B_smem = SMs x 128 B/clk x the SM clock under load."""
    from paper_2305_07390_b200.shapes import get_shape

    mhz = float(sm_mhz) if sm_mhz else 1965.0
    b_smem = sms * SMEM_B_PER_CLK_PER_SM * mhz * 1e6
    a_sm = float(get_shape(stencil).sm_accesses_with_rst)
    bound = b_smem / (a_sm * elem) / 1e9
    return {"bound_gcells": round(bound, 1), "frac": round(gcells / bound, 3),
            "a_sm": a_sm, "b_smem_gbs": round(b_smem / 1e9, 1), "sm_mhz": mhz}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    from oracle import reference_run_threaded
    from paper_2305_07390_b200.rng import uniform_array
    from paper_2305_07390_b200.shapes import make_benchmark

    st = make_benchmark(STENCIL)
    taps = [(tuple(o), c) for o, c in st.taps]
    cells = uniform_array(1, N0 * N1).reshape(N0, N1)
    per_step = max(1, args.ref_tsteps)
    for _ in range(args.warmup):
        reference_run_threaded(cells, taps, 1, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        reference_run_threaded(cells, taps, per_step, threads)
    dt = time.perf_counter() - t0
    gc = (N0 - 2) * (N1 - 2) * per_step * args.steps / dt / 1e9
    sample = (f"{STENCIL} fp64 {N0}x{N1}; each bench step = {per_step} time step(s) of the "
              f"oracle port (numpy, {threads} host threads, axis-0 bands)")
    line = {
        "impl": "reference", "metric": "GCells/s (fp64)", "value": gc, "unit": "GCells/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{STENCIL} fp64 {N0}x{N1} Jacobi sweep (BASELINE config 2)",
                   "time_steps_per_bench_step": per_step, "host_threads": threads},
        "cpu_baseline": {"value": gc, "unit": "GCells/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": gc, "unit": "GCells/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


FP64_LANES_PER_SM = 64  # DP results per clock per SM (tools/dp_microbench.cu, B200)


def _dp_ceiling_gcells(ntaps: int, sms: int, mhz: float) -> float:
    """FP64-pipe ceiling for the shared-product kernels: ntaps DP operations
    per computed cell-step ((ntaps-1) DADD + 1 DMUL), before the valid
    fraction of the tiling."""
    return sms * FP64_LANES_PER_SM * mhz * 1e6 / ntaps / 1e9


def _timed_sweep(device, torch, d_in, st, steps, out, scr, **kw):
    device.sweep_device(d_in, st, steps, out=out, scratch=scr, **kw)  # warm
    torch.cuda.synchronize()
    best = None
    for _ in range(2):
        _, tr = device.sweep_device(d_in, st, steps, out=out, scratch=scr, trace=True, **kw)
        if best is None or tr["elapsed_ms"] < best["elapsed_ms"]:
            best = tr
    return best


def extra_configs(eb, device, _native, torch, stream, hbm_peak):
    """The other BASELINE configs, each on its own synthetic grid (SplitMix64
    seed 1, generated in HBM, exact mode), device-timed with CUDA events:
    config 4 (3-D, 512^3, 500 steps) with its depth sweep, config 3 (large
    halos at 8192^2: overlapped tiling vs halo exchange), the naive
    one-launch-per-step yardstick."""
    try:
        mhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
    except Exception:
        mhz = 1965.0
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = {}

    def rec(name, st, ext, steps, tr, **extra):
        interior = 1
        for n in ext:
            interior *= n - 2 * st.radius
        g = interior * steps / (tr["elapsed_ms"] / 1e3) / 1e9
        r = {"stencil": st.name, "extents": list(ext), "time_steps": steps,
             "value": round(g, 1), "unit": "GCells/s", "ms_per_sweep": round(tr["elapsed_ms"], 3),
             "fused_depth_t": tr["t_used"], "kernel": tr["kernel"],
             "kernel_launches": tr["kernel_launches"], "exact": True,
             "naive_roofline_frac": round(16 * g / hbm_peak, 3),
             "fp64_pipe_ceiling_gcells": round(_dp_ceiling_gcells(len(st.taps), sms, mhz), 1),
             "valid_fraction": round(tr["cells_valid"] / max(1, tr["cells_computed"]), 3),
             "ptb": ptb_fraction(st.name, g, mhz, sms, 4 if extra.get("dtype") == "f32" else 8)}
        r.update(extra)
        out[name] = r

    # ---- config 4: j3d7pt / j3d27pt 512^3, 500 steps ------------------------
    ext3 = (512, 512, 512)
    d3 = device.random_grid_device(ext3, seed=1)
    o3 = torch.empty_like(d3)
    s3 = torch.empty_like(d3)
    st3 = eb.make_benchmark("j3d7pt")
    tr = _timed_sweep(device, torch, d3, st3, 500, o3, s3)
    sweep = {}
    for t in (1, 2, 3, 4):
        tt = _timed_sweep(device, torch, d3, st3, 96, o3, s3, t=t)
        sweep[t] = round((510 ** 3) * 96 / (tt["elapsed_ms"] / 1e3) / 1e9, 1)
    rec("config4_j3d7pt_512", st3, ext3, 500, tr, depth_sweep_gcells=sweep)
    st27 = eb.make_benchmark("j3d27pt")
    tr = _timed_sweep(device, torch, d3, st27, 500, o3, s3)
    rec("config4_j3d27pt_512", st27, ext3, 500, tr)
    # tolerance mode (north star: 1e-12 relative; exact = 0): reassociated sums
    for st_t in (st3, st27):
        tr = _timed_sweep(device, torch, d3, st_t, 500, o3, s3, exact=False)
        rec(f"config4_{st_t.name}_512_tol", st_t, ext3, 500, tr, arith=tr["arith"])
        out[f"config4_{st_t.name}_512_tol"]["exact"] = False
    d3f = d3.float()
    del d3, o3, s3
    torch.cuda.empty_cache()
    o3f = torch.empty_like(d3f)
    s3f = torch.empty_like(d3f)
    tr = _timed_sweep(device, torch, d3f, st3, 500, o3f, s3f)
    rec("config4_j3d7pt_512_fp32", st3, ext3, 500, tr, dtype="f32")
    out["config4_j3d7pt_512_fp32"]["naive_roofline_frac"] = round(
        8 * out["config4_j3d7pt_512_fp32"]["value"] / hbm_peak, 3)
    del d3f, o3f, s3f
    torch.cuda.empty_cache()

    # ---- config 5 geometry on one GPU: j3d7pt 1024^3 (the per-rank slab of
    # the weak-scaling runs), 100 steps -------------------------------------
    ext5 = (1024, 1024, 1024)
    d5 = device.random_grid_device(ext5, seed=1)
    o5 = torch.empty_like(d5)
    s5 = torch.empty_like(d5)
    tr = _timed_sweep(device, torch, d5, st3, 100, o5, s5)
    rec("config5_j3d7pt_1024_1gpu", st3, ext5, 100, tr)
    del d5, o5, s5
    torch.cuda.empty_cache()

    # ---- config 3: large halos at 8192^2, overlapped vs halo exchange -------
    ext2 = (8192, 8192)
    d2 = device.random_grid_device(ext2, seed=1)
    o2 = torch.empty_like(d2)
    s2 = torch.empty_like(d2)
    for name, depths in (("j2d13pt", (2, 3)), ("j2ds25pt", (1, 2))):
        st = eb.get_shape(name)
        for scheme, tag in ((_native.SCHEME_SM_TILING, "overlapped"),
                            (_native.SCHEME_DEVICE_TILING, "halo_exchange")):
            best = None
            for t in depths:
                tr = _timed_sweep(device, torch, d2, st, 96, o2, s2, t=t, scheme=scheme)
                if best is None or tr["elapsed_ms"] < best["elapsed_ms"]:
                    best = tr
            rec(f"config3_{name}_8192_{tag}", st, ext2, 96, best, scheme=tag,
                cluster_ctas=best.get("cluster_ctas", 1))
        # device tiles of several CTAs (cluster halo exchange through DSMEM):
        # the best cluster size of 2/4/8 at the best depth above
        t_h = out[f"config3_{name}_8192_halo_exchange"]["fused_depth_t"]
        best = None
        for cl in (2, 4, 8):
            prm = _native.make_params(scheme=_native.SCHEME_DEVICE_TILING, t=t_h,
                                      device_tile_grid=(1, cl))
            tr = _timed_sweep(device, torch, d2, st, 96, o2, s2, params=prm)
            if best is None or tr["elapsed_ms"] < best["elapsed_ms"]:
                best = tr
        rec(f"config3_{name}_8192_halo_exchange_cluster", st, ext2, 96, best,
            scheme="halo_exchange", cluster_ctas=best["cluster_ctas"])
        # tolerance mode (reassociated sliding sums), planner's default scheme
        tr = _timed_sweep(device, torch, d2, st, 96, o2, s2, exact=False)
        rec(f"config3_{name}_8192_tol", st, ext2, 96, tr, arith=tr["arith"])
        out[f"config3_{name}_8192_tol"]["exact"] = False
    # fp32 mode (north-star 1e-5 tolerance): configs 2 and 4 in binary32;
    # the naive roofline is then 8 B per cell-step
    st5 = eb.make_benchmark("j2d5pt")
    d2f = d2.float()
    o2f = torch.empty_like(d2f)
    s2f = torch.empty_like(d2f)
    tr = _timed_sweep(device, torch, d2f, st5, 1000, o2f, s2f)
    rec("config2_j2d5pt_8192_fp32", st5, ext2, 1000, tr, dtype="f32")
    out["config2_j2d5pt_8192_fp32"]["naive_roofline_frac"] = round(
        8 * out["config2_j2d5pt_8192_fp32"]["value"] / hbm_peak, 3)
    del d2f, o2f, s2f
    # naive yardstick: one launch per time step
    tr = _timed_sweep(device, torch, d2, st5, 20, o2, s2, scheme=_native.SCHEME_NAIVE)
    rec("naive_j2d5pt_8192", st5, ext2, 20, tr)
    del d2, o2, s2
    torch.cuda.empty_cache()
    # 1-D (catalog j1d3pt, its default domain x4): the resident-tile kernel
    # for tap sets without a specialised kernel vs one launch per step
    st1 = eb.make_benchmark("j1d3pt")
    ext1 = (4 * 8388608,)
    d1 = device.random_grid_device(ext1, seed=1)
    o1 = torch.empty_like(d1)
    s1 = torch.empty_like(d1)
    tr = _timed_sweep(device, torch, d1, st1, 256, o1, s1)
    rec("j1d3pt_33554432_resident", st1, ext1, 256, tr)
    tr = _timed_sweep(device, torch, d1, st1, 64, o1, s1, scheme=_native.SCHEME_NAIVE)
    rec("j1d3pt_33554432_naive", st1, ext1, 64, tr)
    del d1, o1, s1
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--t", type=int, default=DEPTH, help="fused depth per HBM round trip")
    ap.add_argument("--tsteps", type=int, default=TSTEPS, help="time steps per bench step")
    ap.add_argument("--ref-tsteps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-3d", action="store_true", help="skip the config-4 3-D measurement")
    ap.add_argument("--no-sweep", action="store_true", help="skip the config-2 t=1..16 sweep")
    ap.add_argument("--no-traffic", action="store_true",
                    help="skip the in-run ncu DRAM-traffic measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch

    import paper_2305_07390_b200 as eb
    from paper_2305_07390_b200 import _native, device

    rank, world, local = dist_env()
    # (local % device_count: the single-GPU multi-rank smoke run of this path,
    # EBISU_BENCH_BACKEND=gloo; one GPU per rank otherwise)
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    backend = os.environ.get("EBISU_BENCH_BACKEND", "nccl")
    red_dev = "cuda" if backend == "nccl" else "cpu"  # gloo reduces host tensors
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            # NCCL's init log (communicator rank count, transports: NVLink P2P /
            # NVLS) lets the run's log prove every rank joined; INIT only, so
            # the JSON result line stays the last line rank 0 prints
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    lib = _native.load()  # fails loudly without the native library
    st = eb.make_benchmark(STENCIL)
    stream = torch.cuda.current_stream()

    if world > 1:
        from paper_2305_07390_b200 import distributed as edist

        # weak scaling: every rank owns an N0 x N1 slab of a (world*N0) x N1 grid
        runner = edist.SlabSweep(st, (N0 * world, N1), t=args.t, seed=1, exact=True)
        step = lambda: runner.run(args.tsteps)  # noqa: E731
        cells_per_step = runner.global_interior_cells() * args.tsteps
        launches_per_step = None  # counted by the runner over the timed region
    else:
        d_in = device.random_grid_device((N0, N1), seed=1)
        d_out = torch.empty_like(d_in)
        d_scr = torch.empty_like(d_in)
        _, tr = device.sweep_device(d_in, st, args.tsteps, out=d_out, scratch=d_scr, t=args.t,
                                    trace=True)
        launches_per_step = tr["kernel_launches"]
        kernel = tr["kernel"]

        def step():
            device.sweep_device(d_in, st, args.tsteps, out=d_out, scratch=d_scr, t=args.t)

        cells_per_step = (N0 - 2) * (N1 - 2) * args.tsteps

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = runner.kernel_launches if world > 1 else 0
    if dist:
        dist.barrier()
    sampler = ClockSampler(dev)
    sampler.start()
    time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    per_launch = []
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        per_launch.append((a, b))
    ev1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1)
    ms_t = torch.tensor([ms], device=red_dev)
    if dist:
        dist.barrier()
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    step_ms = [a.elapsed_time(b) for a, b in per_launch]
    value = cells_per_step * args.steps / (ms / 1e3) / 1e9  # whole job (all ranks)

    hbm_peak, peak_kind = _peaks()
    # dominant kernel: one stream2d_tb launch per bench step when tsteps % t == 0
    # (persistent cooperative launch, grid.sync between epochs)
    launch_ms = statistics.mean(step_ms)
    achieved = ALG_BYTES_PER_CELL_STEP * cells_per_step / world / (launch_ms / 1e3) / 1e9
    traffic, traffic_src = None, None
    if world == 1 and not args.no_traffic:
        traffic, traffic_src = measure_dram_traffic(args.tsteps, args.t)

    line = {
        "metric": "GCells/s (fp64)", "value": value, "unit": "GCells/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SplitMix64 seed 1, generated in HBM)",
        "config": {"workload": f"{STENCIL} fp64 {N0}x{N1}, {args.tsteps} time steps per bench "
                               f"step (BASELINE config 2)",
                   "stencil": STENCIL, "extents": [N0, N1], "time_steps": args.tsteps,
                   "fused_depth_t": args.t, "exact": True,
                   "l2": "inputs larger than L2 (512 MiB grid vs 126 MB L2)",
                   "parallelism": f"slab{world}" if world > 1 else "single",
                   "exchange_every_epochs": runner.exchange_every if world > 1 else None},
        "roofline": {"bound": "hbm", "kernel": "k_stream2d (stream2d_tb)",
                     "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                     "algorithmic_bytes": "16 B per interior cell-step (naive load+store)",
                     "algorithmic_bytes_per_launch": ALG_BYTES_PER_CELL_STEP * cells_per_step
                     // world},
        "ptb": ptb_fraction(STENCIL, value / world, clocks.get("sm_mhz")),
        "clocks": clocks,
        "gpu_launches": (launches_per_step * args.steps) if launches_per_step
        else (runner.kernel_launches - launches0 if world > 1 else None),
    }
    if world == 1:
        line["kernel"] = kernel

    if world == 1 and not args.no_e2e:
        # public C-ABI host call with pinned host buffers; copies inside the region
        host_in = torch.empty((N0, N1), dtype=torch.float64).pin_memory()
        host_out = torch.empty((N0, N1), dtype=torch.float64).pin_memory()
        host_in.copy_(d_in.cpu())
        hin, hout = host_in.numpy(), host_out.numpy()
        import ctypes

        sargs = _native.StencilArgs(st)
        ext = _native.extents_c((N0, N1))
        prm = _native.make_params(t=args.t)

        def e2e_step():
            rc = lib.ebisu_run_host(ctypes.byref(sargs.c), 2, ext, hin.ctypes.data,
                                    hout.ctypes.data, args.tsteps, ctypes.byref(prm), None)
            if rc:
                raise RuntimeError(_native.last_error())

        e2e_step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        dt = time.perf_counter() - t0
        line["e2e"] = {"value": cells_per_step * args.steps / dt / 1e9, "unit": "GCells/s",
                       "h2d_bytes_per_step": N0 * N1 * 8, "d2h_bytes_per_step": N0 * N1 * 8,
                       "api": "ebisu_run_host (pinned host buffers)"}
        # the drop-in Python call a reference user makes: reference_run(Grid,
        # stencil, t) on a pageable numpy grid (grid.py:106-113 signature)
        g_host = eb.Grid(hin.copy(), "fixed-value")
        eb.reference_run(g_host, st, args.tsteps)
        t0 = time.perf_counter()
        nref = 2
        for _ in range(nref):
            eb.reference_run(g_host, st, args.tsteps)
        dt = time.perf_counter() - t0
        line["e2e_reference_run"] = {
            "value": cells_per_step * nref / dt / 1e9, "unit": "GCells/s",
            "h2d_bytes_per_step": N0 * N1 * 8, "d2h_bytes_per_step": N0 * N1 * 8,
            "api": "paper_2305_07390_b200.reference_run (pageable numpy Grid)", "calls": nref}

    if not args.no_sweep and world == 1:
        sweep = {}
        for t in range(1, 17):
            device.sweep_device(d_in, st, 96, out=d_out, scratch=d_scr, t=t)
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            nt = 240 if t <= 8 else 16 * 15
            a.record(stream)
            device.sweep_device(d_in, st, nt, out=d_out, scratch=d_scr, t=t)
            b.record(stream)
            torch.cuda.synchronize()
            sweep[t] = round((N0 - 2) * (N1 - 2) * nt / (a.elapsed_time(b) / 1e3) / 1e9, 1)
        line["depth_sweep_gcells"] = sweep
        # naive yardstick (one launch per step)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        device.sweep_device(d_in, st, 20, out=d_out, scratch=d_scr, scheme=_native.SCHEME_NAIVE)
        b.record(stream)
        torch.cuda.synchronize()
        line["naive_gcells"] = round((N0 - 2) * (N1 - 2) * 20 / (a.elapsed_time(b) / 1e3) / 1e9,
                                     1)

    if world == 1 and not args.no_3d:
        line["configs"] = extra_configs(eb, device, _native, torch, stream, hbm_peak)
        c4 = line["configs"]["config4_j3d7pt_512"]
        line["config4_j3d7pt_512"] = c4  # (kept for round-1 readers)

    if world > 1 and not args.no_3d:
        # BASELINE config 5: j3d7pt fp64, 1024^3 per rank stacked on axis 0
        # (weak scaling) and 1024^3 in total (strong scaling), slab-partitioned
        # with the overlapped NCCL exchange; device time, max over ranks.
        # Guarded: a failure here is reported in the line instead of losing the
        # headline measurement.
        def config5(extents, key, scaling):
            try:
                st3 = eb.make_benchmark("j3d7pt")
                run3 = edist.SlabSweep(st3, extents, t=4, seed=1, exact=True)
                run3.run(8)  # warm-up (2 epochs)
                torch.cuda.synchronize()
                dist.barrier()
                a3 = torch.cuda.Event(enable_timing=True)
                b3 = torch.cuda.Event(enable_timing=True)
                a3.record(stream)
                run3.run(100)
                b3.record(stream)
                torch.cuda.synchronize()
                t3 = torch.tensor([a3.elapsed_time(b3)], device=red_dev)
                dist.all_reduce(t3, op=dist.ReduceOp.MAX)
                ms3 = float(t3.item())
                cells3 = run3.global_interior_cells() * 100
                line[key] = {
                    "value": cells3 / (ms3 / 1e3) / 1e9, "unit": "GCells/s", "ms": ms3,
                    "time_steps": 100, "fused_depth_t": 4, "scaling": scaling,
                    "extents": list(extents), "overlapped_epochs": run3.overlapped_epochs,
                    "exchange_every_epochs": run3.exchange_every}
                del run3
                torch.cuda.empty_cache()
            except Exception as exc:  # pragma: no cover - multi-GPU only
                line[key] = {"error": repr(exc)[:300]}

        config5((1024 * world, 1024, 1024), "config5_weak_j3d7pt_1024_per_rank", "weak")
        config5((1024, 1024, 1024), "config5_strong_j3d7pt_1024_total", "strong")

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_oracle_sample()
    if rank == 0:
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
