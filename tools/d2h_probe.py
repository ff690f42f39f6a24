"""Host-side limits of a full W download (development aid): pinned D2H bandwidth,
first-touch cost of a fresh numpy buffer, and cudaHostRegister of a fresh buffer."""
import time

import numpy as np
import torch

n = 5 << 30
d = torch.empty(n // 8, dtype=torch.float64, device="cuda")
h = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); h.copy_(d, non_blocking=True); torch.cuda.synchronize()
    print(f"pinned D2H {n / (time.perf_counter() - t0) / 1e9:.1f} GB/s", flush=True)
cr = torch.cuda.cudart()
for chunk in (n, 256 << 20, 64 << 20):
    a = np.empty(n // 8)
    t0 = time.perf_counter()
    base = a.ctypes.data
    for off in range(0, n, chunk):
        assert int(cr.cudaHostRegister(base + off, min(chunk, n - off), 0)) == 0
    t1 = time.perf_counter()
    ta = torch.from_numpy(a)
    ta.copy_(d, non_blocking=True); torch.cuda.synchronize()
    t2 = time.perf_counter()
    for off in range(0, n, chunk):
        cr.cudaHostUnregister(base + off)
    t3 = time.perf_counter()
    print(f"chunk {chunk >> 20} MB: register {n / (t1 - t0) / 1e9:.1f} GB/s, DMA into registered {n / (t2 - t1) / 1e9:.1f} GB/s,"
          f" unregister {1e3 * (t3 - t2):.1f} ms", flush=True)
