"""Multi-rank slab decomposition on CPU with the gloo backend.

The exchange plan and epoch loop of paper_2305_07390_b200.distributed run
exactly as on GPUs; only the per-rank compute is injected from the oracle
(tests may use the oracle as checker/stand-in; the product default is the
CUDA kernel).  The gathered result must be bitwise equal to the oracle's
full-grid reference_run.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import taps_of


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = [
    ("j2d5pt", (40, 30), 7, 3),
    ("j2d9pt", (50, 20), 6, 2),
    ("j2d25pt", (37, 18), 5, 2),
    ("j3d7pt", (24, 10, 12), 5, 2),
    ("j3d27pt", (21, 9, 8), 4, 3),
    ("j2d5pt", (64, 16), 9, 4),
]


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import reference_run
        import paper_2305_07390_b200 as eb
        from paper_2305_07390_b200.distributed import SlabSweep

        out = {}
        for i, (name, ext, steps, t) in enumerate(CASES):
            st = eb.get_shape(name)
            taps = taps_of(st)

            def step(src, dst, scratch, n, _t, planes=None, frame_ready=False, taps=taps):
                # same contract as the kernel: ``planes`` restricts the planes
                # written (ebisu_params.out_planes); the rest of dst is untouched
                res = torch.from_numpy(reference_run(src.numpy(), taps, n))
                if planes is None:
                    dst.copy_(res)
                else:
                    dst[planes[0]:planes[1]].copy_(res[planes[0]:planes[1]])

            sw = SlabSweep(st, ext, t=t, seed=1000 + i, step=step, device=torch.device("cpu"),
                           exchange_every=1)
            sw.run(steps)
            own_n = sw.plan.own1 - sw.plan.own0
            if own_n >= 2 * sw.halo and steps >= t:
                assert sw.overlapped_epochs == steps // t, (name, sw.overlapped_epochs)
            full = sw.gather(0)
            if rank == 0:
                out[i] = full.numpy()
            # deep halos: K epochs per exchange, one sweep of the whole local
            # slab (ghosts included) per K epochs
            for k in (2, 3):
                if (ext[0] // world) < 2 * k * t * st.radius:
                    continue
                sw = SlabSweep(st, ext, t=t, seed=1000 + i, step=step,
                               device=torch.device("cpu"), exchange_every=k)
                sw.run(steps)
                full = sw.gather(0)
                if rank == 0:
                    out[(i, k)] = full.numpy()
        if rank == 0:
            results.update(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_sweep_matches_oracle(world):
    from oracle import reference_run
    import paper_2305_07390_b200 as eb

    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    for i, (name, ext, steps, t) in enumerate(CASES):
        st = eb.get_shape(name)
        g = eb.random_grid(ext, 1000 + i)
        ref = reference_run(g.cells, taps_of(st), steps)
        assert np.array_equal(results[i], ref), (world, name, ext, steps, t)
        for k in (2, 3):
            if (i, k) in results:
                assert np.array_equal(results[(i, k)], ref), (world, name, ext, steps, t, k)
    assert any(isinstance(key, tuple) for key in results.keys())  # deep mode exercised


def test_slab_plan_geometry():
    from paper_2305_07390_b200.distributed import slab_plan

    plans = [slab_plan(103, 4, r, 6) for r in range(4)]
    assert plans[0].own0 == 0 and plans[-1].own1 == 103
    assert all(a.own1 == b.own0 for a, b in zip(plans, plans[1:]))
    assert plans[0].ghost_lo == 0 and plans[-1].ghost_hi == 0
    assert all(p.ghost_lo == 6 for p in plans[1:]) and all(p.ghost_hi == 6 for p in plans[:-1])
    with pytest.raises(ValueError, match="thinner"):
        slab_plan(10, 4, 0, 6)


def _gpu_worker(rank, world, port, results):
    """Two ranks on one GPU: the real CUDA step (ranged band/interior kernel
    calls, comm stream) with gloo host-staged P2P standing in for NCCL."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2305_07390_b200 as eb
        from paper_2305_07390_b200.distributed import SlabSweep

        out = {}
        for i, (name, ext, steps, t) in enumerate(GPU_CASES):
            st = eb.get_shape(name)
            sw = SlabSweep(st, ext, t=t, seed=2000 + i, device=torch.device("cuda", 0),
                           exchange_every=1)
            sw.run(steps)
            torch.cuda.synchronize()
            full = sw.gather(0)
            if rank == 0:
                out[i] = (full.numpy(), sw.overlapped_epochs)
            # deep halos (2 epochs per exchange, one persistent sweep each)
            if ext[0] // world >= 4 * t * st.radius:
                sw = SlabSweep(st, ext, t=t, seed=2000 + i, device=torch.device("cuda", 0),
                               exchange_every=2)
                sw.run(steps)
                torch.cuda.synchronize()
                full = sw.gather(0)
                if rank == 0:
                    out[(i, 2)] = full.numpy()
        if rank == 0:
            results.update(out)
    finally:
        dist.destroy_process_group()


GPU_CASES = [
    ("j2d5pt", (300, 260), 17, 8),
    ("j3d7pt", (70, 40, 66), 9, 4),
    ("j3d27pt", (44, 30, 34), 5, 2),
    ("j2ds25pt", (200, 264), 3, 1),
]


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_slab_sweep_gpu_kernels(world):
    """The multi-GPU epoch loop with the GPU kernels (band-first ranged calls,
    interior on the compute stream, exchange on the comm stream) equals the
    single-grid oracle bitwise."""
    from oracle import reference_run
    import paper_2305_07390_b200 as eb

    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_gpu_worker, args=(world, port, results), nprocs=world, join=True)
    for i, (name, ext, steps, t) in enumerate(GPU_CASES):
        st = eb.get_shape(name)
        g = eb.random_grid(ext, 2000 + i)
        ref = reference_run(g.cells, taps_of(st), steps)
        got, overlapped = results[i]
        assert np.array_equal(got, ref), (world, name, ext, steps, t)
        assert overlapped == steps // t, (name, overlapped)
        if (i, 2) in results:
            assert np.array_equal(results[(i, 2)], ref), (world, name, "deep halo")
    assert any(isinstance(key, tuple) for key in results.keys())
