"""Host<->device copy strategies for pageable numpy buffers (512 MiB each way)."""
import ctypes, time, os, sys, threading
import numpy as np
import torch
n = 8192 * 8192
src = np.random.rand(n)
dst = np.empty_like(src)
d = torch.empty(n, dtype=torch.float64, device="cuda")
cud = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
print("cudart", cud)
def tm(f, reps=3):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
ts = torch.from_numpy(src); tdst = torch.from_numpy(dst)
print("pageable h2d ms", tm(lambda: d.copy_(ts)))
print("pageable d2h ms", tm(lambda: tdst.copy_(d)))
pin = torch.empty(n, dtype=torch.float64).pin_memory()
print("pinned h2d ms", tm(lambda: d.copy_(pin, non_blocking=True)))
print("pinned d2h ms", tm(lambda: pin.copy_(d, non_blocking=True)))
cudart = torch.cuda.cudart()
def reg():
    r = cudart.cudaHostRegister(src.ctypes.data, src.nbytes, 0)
    d.copy_(ts, non_blocking=True); torch.cuda.synchronize()
    cudart.cudaHostUnregister(src.ctypes.data)
print("register+h2d+unregister ms", tm(reg))
def regonly():
    cudart.cudaHostRegister(src.ctypes.data, src.nbytes, 0)
    cudart.cudaHostUnregister(src.ctypes.data)
print("register+unregister ms", tm(regonly))
# staged: T threads memcpy chunks into pinned ring, main issues async copies
def staged(nthreads=8, chunk=1 << 24):
    nb = src.nbytes
    ring = [torch.empty(chunk // 8, dtype=torch.float64).pin_memory() for _ in range(2 * nthreads)]
    s = torch.cuda.Stream()
    evs = [None] * len(ring)
    off = 0; k = 0
    sv = memoryview(src).cast("B")
    with torch.cuda.stream(s):
        chunks = [(o, min(chunk, nb - o)) for o in range(0, nb, chunk)]
        i = 0
        while i < len(chunks):
            batch = chunks[i:i + nthreads]
            th = []
            for j, (o, ln) in enumerate(batch):
                slot = (i + j) % len(ring)
                if evs[slot] is not None: evs[slot].synchronize()
                def cp(slot=slot, o=o, ln=ln):
                    ctypes.memmove(ring[slot].data_ptr(), src.ctypes.data + o, ln)
                t = threading.Thread(target=cp); t.start(); th.append((t, slot, o, ln))
            for t, slot, o, ln in th:
                t.join()
                d.view(torch.uint8)[o:o + ln].copy_(ring[slot].view(torch.uint8)[:ln], non_blocking=True)
                e = torch.cuda.Event(); e.record(s); evs[slot] = e
            i += nthreads
    s.synchronize()
print("staged 8 threads h2d ms", tm(staged))
print("host memcpy 512MB 1 thread ms", tm(lambda: ctypes.memmove(dst.ctypes.data, src.ctypes.data, src.nbytes)))
print("cpus", os.cpu_count())
