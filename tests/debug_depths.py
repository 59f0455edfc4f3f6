"""Debug helper (not collected by pytest): run each fused depth in its own
process and report pass/fail against the oracle."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2305_07390_b200 as eb
from oracle import reference_run
name, t, n0, n1, steps, pers = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), int(sys.argv[6])
st = eb.get_shape(name)
g = eb.random_grid((n0, n1), 5)
out, tr = eb.sweep(g, st, steps, t=t, persistent=bool(pers), trace=True)
ref = reference_run(g.cells, [(tuple(o), c) for o, c in st.taps], steps)
ok = np.array_equal(out.cells, ref)
print("OK" if ok else "MISMATCH", tr["kernel"], tr["kernel_launches"], np.abs(out.cells-ref).max())
''' % ROOT
cases = [a.split(",") for a in sys.argv[1:]] or [["j2d5pt", str(t), "200", "260", str(3 * t + 1), "1"] for t in range(1, 17)]
for c in cases:
    r = subprocess.run([sys.executable, "-c", CODE] + c, capture_output=True, text=True, timeout=120,
                       env=dict(os.environ, CUDA_LAUNCH_BLOCKING="1"))
    msg = (r.stdout.strip() or r.stderr.strip().splitlines()[-1:] or ["?"])
    print(",".join(c), "->", msg if isinstance(msg, str) else msg[0], flush=True)
