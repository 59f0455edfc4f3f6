"""bench.py contract checks that run without a GPU: the reference arm's JSON
line (oracle port on the host) and the argument surface."""

from __future__ import annotations

import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    env = dict(os.environ, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "3", "--ref-tsteps", "1"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == "GCells/s (fp64)" and d["unit"] == "GCells/s"
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["warmup"] >= 3


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, PYTHONPATH=ROOT, RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference"],
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


import pytest  # noqa: E402


@pytest.mark.gpu
def test_ours_arm_json_line():
    """The GPU arm's line (short sweep): contract keys, roofline and e2e."""
    env = dict(os.environ, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2",
                        "--warmup", "3", "--tsteps", "64", "--no-3d", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "clocks", "gpu_launches", "e2e"):
        assert key in d, key
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["warmup"] >= 3
    assert d["roofline"]["peak"] > 0 and d["roofline"]["frac"] > 0
    assert d["gpu_launches"] >= d["steps"]
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["kernel"] == "stream2d_tb"


@pytest.mark.gpu
def test_multi_rank_bench_path_on_one_gpu():
    """The N>1 bench path (torchrun, slab decomposition, overlapped epochs,
    max-over-ranks timing, config-5 line) end to end: two ranks share one GPU
    with gloo standing in for NCCL (EBISU_BENCH_BACKEND=gloo)."""
    env = dict(os.environ, PYTHONPATH=ROOT, EBISU_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", "29517", os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "1", "--warmup", "3", "--tsteps", "16"],
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "weak"
    assert d["gpu_launches"] > 0
    for key in ("config5_weak_j3d7pt_1024_per_rank", "config5_strong_j3d7pt_1024_total"):
        c5 = d[key]
        # per-epoch overlapped split, or deep halos (K epochs per exchange)
        assert "error" not in c5 and c5["value"] > 0, c5
        assert c5["overlapped_epochs"] > 0 or c5["exchange_every_epochs"] > 1, c5
