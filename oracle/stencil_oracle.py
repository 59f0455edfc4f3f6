"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference Jacobi sweep.

Restates ``stencilplan.grid`` (reference ``pkg/src/stencilplan/grid.py``) and
``stencilplan.rng.uniform_array`` (``rng.py:31-46``) over plain ndarrays and
``((offset...), coeff)`` tap lists, so it shares no code with the product
package.  Used by ``tests/`` (checker), ``__graft_entry__.smoke()`` (checker)
and ``bench.py`` (CPU baseline / ``--impl reference``) only.

Arithmetic contract (what the GPU exact mode must reproduce): per interior
cell, ``acc = c0*x[o0]`` then ``acc = acc + ck*x[ok]`` for k = 1.. in tap
order, every multiply and add a separately rounded IEEE binary64 operation
(numpy ufuncs never contract to FMA).  Frame cells (distance < radius from any
face) keep their input value.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

_MASK = (1 << 64) - 1


def uniform_array(seed: int, n: int) -> np.ndarray:
    """First ``n`` uniforms of SplitMix64(seed) -- reference ``rng.py:31-46``."""
    idx = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & _MASK) + idx * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def _radius(taps) -> int:
    return max(abs(c) for off, _ in taps for c in off)


def check_compatible(cells: np.ndarray, taps, name: str = "stencil"):
    """Reference ``grid.py:63-73`` (same messages)."""
    dims = len(taps[0][0])
    if cells.ndim != dims:
        raise ValueError(f"grid is {cells.ndim}-D but stencil {name} is {dims}-D")
    rad = _radius(taps)
    for n in cells.shape:
        if n <= 2 * rad:
            raise ValueError(f"extent {n} too small for radius {rad} (need > {2 * rad})")


def apply_taps(cells: np.ndarray, taps, rows=None) -> np.ndarray:
    """Interior tap sum in tap order -- reference ``grid.py:76-93``.

    ``rows=(a, b)`` restricts the result to interior rows ``a..b-1`` of axis 0
    (absolute indices); the per-cell operation sequence is unchanged, which is
    what makes the banded/threaded sweep bitwise equal to the whole-array one.
    """
    rad = _radius(taps)
    shape = cells.shape
    a, b = (rad, shape[0] - rad) if rows is None else rows
    acc = None
    for off, c in taps:
        sl = (slice(a + off[0], b + off[0]),) + tuple(
            slice(rad + o, n - rad + o) for o, n in zip(off[1:], shape[1:])
        )
        term = c * cells[sl]
        acc = term if acc is None else acc + term
    return acc


def reference_step(cells: np.ndarray, taps) -> np.ndarray:
    """One Jacobi step, pure -- reference ``grid.py:96-103``."""
    check_compatible(cells, taps)
    rad = _radius(taps)
    out = cells.copy()
    core = tuple(slice(rad, n - rad) for n in cells.shape)
    out[core] = apply_taps(cells, taps)
    return out


def reference_run(cells: np.ndarray, taps, t: int) -> np.ndarray:
    """``t``-fold composition -- reference ``grid.py:106-113``."""
    if t < 0:
        raise ValueError("step count must be >= 0")
    out = np.array(cells, dtype=np.float64, copy=True)
    for _ in range(t):
        out = reference_step(out, taps)
    return out


def reference_run_threaded(cells: np.ndarray, taps, t: int, threads: int) -> np.ndarray:
    """Same sweep with axis-0 interior bands on ``threads`` host threads.

    numpy releases the GIL inside ufunc loops, so bands run concurrently.
    Each output cell sees exactly the operation sequence of ``reference_step``
    (bitwise equal; checked in ``tests/test_oracle.py``).  This is the
    "all host threads" CPU arm of ``bench.py --impl reference``.
    """
    if t < 0:
        raise ValueError("step count must be >= 0")
    cur = np.array(cells, dtype=np.float64, copy=True)
    if t == 0:
        return cur
    check_compatible(cur, taps)
    rad = _radius(taps)
    n0 = cur.shape[0]
    inner = n0 - 2 * rad
    threads = max(1, min(threads, inner))
    bounds = [rad + (inner * i) // threads for i in range(threads + 1)]
    bands = [(bounds[i], bounds[i + 1]) for i in range(threads) if bounds[i + 1] > bounds[i]]
    core_rest = tuple(slice(rad, n - rad) for n in cur.shape[1:])
    with ThreadPoolExecutor(max_workers=len(bands)) as pool:
        for _ in range(t):
            nxt = cur.copy()

            def band(ab, src=cur, dst=nxt):
                a, b = ab
                dst[(slice(a, b),) + core_rest] = apply_taps(src, taps, rows=(a, b))

            list(pool.map(band, bands))
            cur = nxt
    return cur
