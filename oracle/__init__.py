"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the Jacobi sweep.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2305_07390_b200``) never imports, links or executes it; a missing CUDA
extension makes the product raise instead of falling back here.

Parity status: PINNED.  ``tests/golden/make_golden.py`` ran the unmodified
reference (``/root/reference/pkg/src/stencilplan``) in the build container and
committed its outputs (SHA-256 digests plus small arrays) to ``tests/golden/``;
``tests/test_oracle.py`` checks this restatement against every one of them and
against the reference's own known-answer tests (impulse, scalar double loop,
3-D brute force; ``pkg/tests/test_grid.py:33-91``).
"""

from .stencil_oracle import (  # noqa: F401
    apply_taps,
    check_compatible,
    reference_run,
    reference_run_threaded,
    reference_step,
    uniform_array,
)
