"""Multi-GPU sweep: slab decomposition along axis 0.

Not in the reference (it has no distributed backend); this is the
B200 build's scale-out of ``reference_run`` over the GPUs of one node.

* Rank g owns the contiguous planes ``[own0, own1)`` of axis 0 (the streaming
  axis, slowest in C order, so slabs and halos are contiguous blocks).
* Each rank keeps ``H = t*R`` ghost planes on every interior face.  Per epoch
  (t fused steps), overlapped: (1) compute the two boundary bands -- the H
  owned planes next to each interior face, the only outputs a neighbour
  needs -- with the single-GPU kernel restricted to those output planes
  (``ebisu_params.out_planes``); (2) on a communication stream, send the
  bands and receive the neighbours' bands straight into the ghost planes
  (NCCL point-to-point through ``torch.distributed``, one batched group);
  (3) meanwhile compute the interior planes, which need no ghost; (4) join.
  Slabs thinner than 2H, and the remainder epoch of a step count that is not
  a multiple of t, run unsplit and exchange afterwards.  The array faces at ghost boundaries are
  treated as frame by the kernel; the error this introduces travels R planes
  per step, so after t steps it has crossed exactly the H ghost planes and the
  owned planes are exact -- bitwise equal to ``reference_run`` on the full
  grid (tests/test_distributed.py).
* Global frame planes belong to the first/last rank, which have no ghost on
  that face, so the kernel's own frame handling applies there.

The compute step is a parameter only so that the CPU tests can drive the same
exchange logic with the oracle; the product default is the GPU kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

from .shapes import StencilShape


@dataclass(frozen=True)
class SlabPlan:
    """One rank's share of axis 0 (all indices are global plane numbers)."""

    rank: int
    world: int
    n0: int
    own0: int
    own1: int
    ghost_lo: int  # ghost planes below own0 held locally
    ghost_hi: int  # ghost planes above own1 held locally

    @property
    def local0(self) -> int:
        return self.own0 - self.ghost_lo

    @property
    def local1(self) -> int:
        return self.own1 + self.ghost_hi

    @property
    def local_planes(self) -> int:
        return self.local1 - self.local0


def slab_plan(n0: int, world: int, rank: int, halo: int) -> SlabPlan:
    """Even split of ``n0`` planes; ``halo`` ghost planes per interior face."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n0, world)
    own0 = rank * base + min(rank, extra)
    own1 = own0 + base + (1 if rank < extra else 0)
    if world > 1 and base < halo:
        raise ValueError(
            f"slab of {base} planes is thinner than the {halo}-plane halo; "
            "use fewer ranks or a smaller fused depth"
        )
    lo = halo if rank > 0 else 0
    hi = halo if rank < world - 1 else 0
    return SlabPlan(rank, world, n0, own0, own1, lo, hi)


# SMs the interior kernel leaves to NCCL's point-to-point kernels (one or two
# CTAs per channel and peer) -- see SlabSweep.__init__
INTERIOR_RESERVE_SMS = 2


def _default_step(stencil: StencilShape, exact: bool):
    """The per-epoch sweep call of the slab driver.  The epoch loop issues three
    ranged calls per epoch (~0.3 ms of GPU work each at j2d5pt 8192^2 t=8),
    so the host side is kept lean: the stencil arguments, the extents and the
    parameter blocks are built once and reused, and the C ABI is called
    directly on the current stream (same call as device.sweep_device)."""
    import ctypes

    from . import _native, device

    lib = _native.load()
    sargs = _native.StencilArgs(stencil)
    ext_cache: dict = {}
    prm_cache: dict = {}

    def step(src, dst, scratch, steps, t, planes=None, frame_ready=False, reserve_sms=0):
        if planes is None:
            device.sweep_device(src, stencil, steps, out=dst, scratch=scratch, t=t, exact=exact)
            return
        # frame_ready: dst already holds the (constant) frame, so the ranged
        # call skips its frame pre-copy launch; reserve_sms keeps SMs free of
        # the interior grid for the concurrent NCCL kernels
        key = (t, tuple(planes), bool(frame_ready), int(reserve_sms))
        prm = prm_cache.get(key)
        if prm is None:
            prm = prm_cache[key] = _native.make_params(
                t=t, exact=exact, out_planes=planes, frame_ready=frame_ready,
                reserve_sms=reserve_sms)
        shape = tuple(src.shape)
        ext = ext_cache.get(shape)
        if ext is None:
            ext = ext_cache[shape] = _native.extents_c(shape)
        run = lib.ebisu_run_device_f32 if src.dtype == device._torch().float32 else \
            lib.ebisu_run_device
        rc = run(ctypes.byref(sargs.c), src.dim(), ext, src.data_ptr(), dst.data_ptr(), None,
                 int(steps), ctypes.byref(prm), device._stream_ptr(), None)
        if rc:
            raise _native.NativeError(f"libebisu error {rc}: {_native.last_error()}")

    return step


class SlabSweep:
    """Distributed ``reference_run`` over ``torch.distributed`` ranks.

    ``extents`` is the GLOBAL grid shape; each rank allocates only its slab
    plus ghosts.  ``seed`` draws the global SplitMix64 grid, each rank
    generating exactly its own planes (``ebisu_random_grid_device`` with the
    global start offset).
    """

    def __init__(self, stencil: StencilShape, extents, t: int, seed: int | None = None,
                 exact: bool = True, group=None, device=None, step=None, cells=None,
                 exchange_every: int | None = None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.stencil = stencil
        self.extents = tuple(int(n) for n in extents)
        self.t = int(t)
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        # Deep halos: exchange every K epochs with K*t*R ghost planes, the K
        # epochs in ONE persistent sweep of the whole local slab (ghosts
        # included): the slab's own frame planes sit in the ghost region, whose
        # values go stale by R planes per step -- K*t*R planes after K epochs,
        # exactly the ghost depth -- so the owned planes stay exact, and the
        # sweep keeps its dataflow epochs (no epoch tail; the per-epoch
        # band/interior split measured at <= 0.87 of a persistent sweep on one
        # GPU, tools/slab_split_cost.py).  Cost: 2*K*t*R redundant planes per
        # rank.  Default: the largest K <= 16 with that redundancy <= 1.6 % of
        # the owned planes (K = 1: the overlapped per-epoch split).  Measured
        # on one GPU for a middle rank of config 2 (8192^2 per rank, t=8):
        # K = 4 / 8 / 16 -> 0.90 / 0.94 / 0.93 of the owned-only sweep, the
        # per-epoch split 0.86 (profiles/r02_slab_split_cost.txt).
        R = max(1, stencil.radius)
        if exchange_every is None:
            own = self.extents[0] // max(1, self.world)
            exchange_every = int(0.008 * own // (self.t * R)) if self.world > 1 else 1
        self.exchange_every = max(1, min(16, int(exchange_every)))
        self.halo = self.exchange_every * self.t * stencil.radius
        self.plan = slab_plan(self.extents[0], self.world, self.rank, self.halo)
        self.device = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available()
            else torch.device("cpu"))
        self.step = step if step is not None else _default_step(stencil, exact)
        # The interior grid is persistent (one CTA per SM): if it held every
        # SM, the NCCL send/recv kernels of the band exchange (launched on the
        # communication stream behind the band kernels) could not start until
        # the interior finished, and the exchange would serialise behind it.
        # INTERIOR_RESERVE_SMS SMs stay free for them (1.4 % of the interior's
        # throughput at 2 of 148).
        self._interior_kw = {"reserve_sms": INTERIOR_RESERVE_SMS} if step is None else {}
        rest = self.extents[1:]
        shape = (self.plan.local_planes,) + rest
        plane = 1
        for n in rest:
            plane *= n
        self.plane_cells = plane
        if cells is not None:
            a = cells.to(self.device, dtype=torch.float64).contiguous()
            if tuple(a.shape) != shape:
                raise ValueError(f"local slab must have shape {shape}")
        else:
            a = torch.empty(shape, dtype=torch.float64, device=self.device)
            if seed is not None:
                self._fill_random(a, seed)
        self.a = a
        self.b = torch.empty_like(a)
        self.scratch = torch.empty_like(a)
        self.comm = torch.cuda.Stream(self.device) if a.is_cuda else None
        self.overlapped_epochs = 0
        # buffers holding the Dirichlet frame (the input does; an epoch's
        # output does once its ranged calls copied theirs)
        self._framed = {a.data_ptr()}
        # kernels launched by the default step (bench gpu_launches claim): a
        # ranged single-epoch call = frame copy + TB kernel; a full epoch call
        # = two frame copies (out and scratch) + TB kernel
        self.kernel_launches = 0

    # -- data --------------------------------------------------------------
    def _fill_random(self, a, seed: int):
        if a.is_cuda:
            import ctypes  # noqa: F401

            from . import _native, device

            lib = _native.load()
            rc = lib.ebisu_random_grid_device(int(seed) & ((1 << 64) - 1),
                                              self.plan.local0 * self.plane_cells, a.numel(),
                                              a.data_ptr(), device._stream_ptr())
            if rc:
                raise _native.NativeError(_native.last_error())
        else:
            from .rng import uniform_array

            vals = uniform_array(seed, a.numel(), start=self.plan.local0 * self.plane_cells)
            a.copy_(self.torch.from_numpy(vals.reshape(tuple(a.shape))))

    def owned(self):
        """This rank's owned planes of the current state (a view)."""
        p = self.plan
        return self.a[p.ghost_lo:p.ghost_lo + (p.own1 - p.own0)]

    def global_interior_cells(self) -> int:
        r = self.stencil.radius
        n = 1
        for e in self.extents:
            n *= e - 2 * r
        return n

    # -- communication ---------------------------------------------------------
    def _p2p(self, pairs):
        """Batched point-to-point exchange of (send, recv, peer) triples.
        NCCL moves device tensors directly; a backend without device P2P
        (gloo: the single-GPU multi-rank tests) stages them through host
        memory."""
        dist = self.dist
        staged = []
        ops = []
        host = dist.get_backend(self.group) == "gloo"
        for send, recv, peer in pairs:
            if host and send.is_cuda:
                hs, hr = send.cpu(), self.torch.empty(recv.shape, dtype=recv.dtype)
                staged.append((hr, recv))
                send, recv = hs, hr
            ops.append(dist.P2POp(dist.isend, send, peer, self.group))
            ops.append(dist.P2POp(dist.irecv, recv, peer, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for hr, recv in staged:
            recv.copy_(hr)

    def exchange(self, depth: int):
        """Refresh ``depth`` ghost planes on each interior face."""
        if self.world == 1 or depth == 0:
            return
        p = self.plan
        a = self.a
        lo0 = p.ghost_lo
        hi0 = p.ghost_lo + (p.own1 - p.own0)
        pairs = []
        if p.rank > 0:
            pairs.append((a[lo0:lo0 + depth], a[lo0 - depth:lo0], p.rank - 1))
        if p.rank < p.world - 1:
            pairs.append((a[hi0 - depth:hi0], a[hi0:hi0 + depth], p.rank + 1))
        self._p2p(pairs)

    def _bands(self):
        """Local plane ranges: (lower band, upper band, interior) of the owned
        planes; a band is None on a face without neighbour."""
        p, H = self.plan, self.halo
        o0, o1 = p.ghost_lo, p.ghost_lo + (p.own1 - p.own0)
        lo = (o0, o0 + H) if p.rank > 0 else None
        hi = (o1 - H, o1) if p.rank < p.world - 1 else None
        return lo, hi, (o0 + (H if lo else 0), o1 - (H if hi else 0))

    def _exchange_bands(self, dst, lo, hi):
        """Send the freshly computed bands of ``dst``; receive the neighbours'
        bands straight into the ghost planes of ``dst``."""
        p, H = self.plan, self.halo
        pairs = []
        if lo:
            pairs.append((dst[lo[0]:lo[1]], dst[lo[0] - H:lo[0]], p.rank - 1))
        if hi:
            pairs.append((dst[hi[0]:hi[1]], dst[hi[1]:hi[1] + H], p.rank + 1))
        self._p2p(pairs)

    def _epoch_overlapped(self):
        """One t-step epoch.  Communication stream: the two boundary bands,
        then their exchange; compute stream, concurrently: the interior.  The
        bands are launched first so their few CTAs get SMs before the
        interior grid fills the rest; band kernel and exchange both leave the
        critical path (the interior takes longer than either)."""
        t = self.t
        lo, hi, inner = self._bands()
        ready = self.b.data_ptr() in self._framed
        per_call = 1 if ready else 2  # TB kernel (+ frame pre-copy)

        def bands():
            for band in (lo, hi):
                if band:
                    self.step(self.a, self.b, None, t, t, planes=band, frame_ready=ready)
                    self.kernel_launches += per_call

        def interior():
            if inner[1] > inner[0]:
                self.step(self.a, self.b, None, t, t, planes=inner, frame_ready=ready,
                          **self._interior_kw)
                self.kernel_launches += per_call

        if self.comm is not None:
            torch = self.torch
            compute = torch.cuda.current_stream(self.device)
            self.comm.wait_stream(compute)  # previous epoch (and its ghosts) done
            with torch.cuda.stream(self.comm):
                bands()
                self._exchange_bands(self.b, lo, hi)
            interior()
            compute.wait_stream(self.comm)  # ghosts of the next epoch landed
        else:
            bands()
            self._exchange_bands(self.b, lo, hi)
            interior()
        self._framed.add(self.b.data_ptr())
        self.overlapped_epochs += 1

    # -- sweep ------------------------------------------------------------------
    def run(self, steps: int):
        """Advance the distributed grid by ``steps`` Jacobi steps."""
        if steps < 0:
            raise ValueError("step count must be >= 0")
        if steps == 0:
            return self.owned()
        own_n = self.plan.own1 - self.plan.own0
        if self.exchange_every > 1:
            return self._run_deep(steps)
        split = self.world > 1 and own_n >= 2 * self.halo
        self.exchange(self.halo)  # ghosts current from here on
        done = 0
        while done < steps:
            d = min(self.t, steps - done)
            if split and d == self.t:
                self._epoch_overlapped()
            else:
                self.step(self.a, self.b, self.scratch, d, d)
                self.kernel_launches += 3
                self._framed.update((self.b.data_ptr(), self.scratch.data_ptr()))
                self.a, self.b = self.b, self.a
                if done + d < steps:
                    self.exchange(self.halo)
                done += d
                continue
            self.a, self.b = self.b, self.a
            done += d
        return self.owned()

    def _run_deep(self, steps: int):
        """Deep-halo loop: persistent sweeps of K epochs, exchange between."""
        self.exchange(self.halo)
        done = 0
        while done < steps:
            d = min(self.exchange_every * self.t, steps - done)
            self.step(self.a, self.b, self.scratch, d, self.t)
            self.kernel_launches += 3  # TB kernel + frame copies (out, scratch)
            self._framed.update((self.b.data_ptr(), self.scratch.data_ptr()))
            self.a, self.b = self.b, self.a
            done += d
            if done < steps:
                self.exchange(self.halo)
        return self.owned()

    def gather(self, dst: int = 0):
        """Full grid on rank ``dst`` (tests / verification); None elsewhere."""
        torch, dist = self.torch, self.dist
        own = self.owned().contiguous()
        if self.world == 1:
            return own.cpu()
        sizes = [slab_plan(self.extents[0], self.world, r, self.halo) for r in range(self.world)]
        # gloo has no device P2P: stage through host memory (tests)
        dev = "cpu" if dist.get_backend(self.group) == "gloo" else own.device
        if self.rank == dst:
            parts = []
            for r, pr in enumerate(sizes):
                if r == dst:
                    parts.append(own.cpu())
                else:
                    buf = torch.empty((pr.own1 - pr.own0,) + self.extents[1:],
                                      dtype=own.dtype, device=dev)
                    dist.recv(buf, src=r, group=self.group)
                    parts.append(buf.cpu())
            return torch.cat(parts, 0)
        dist.send(own.to(dev), dst=dst, group=self.group)
        return None
