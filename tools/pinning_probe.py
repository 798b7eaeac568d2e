"""Host->device of a caller's pageable numpy fp64 array (the drop-in GradientState input), 2.68 GB:
pageable copy vs cudaHostRegister + async copy (+ unregister) vs a pinned staging ring fed by
host threads.  Prints one JSON line."""
import json
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

D = 335_141_888
a = np.random.default_rng(0).standard_normal(D)  # fp64, pageable
dev = torch.empty(D, dtype=torch.float64, device="cuda")
res = {}
torch.cuda.synchronize()
t = time.perf_counter()
dev.copy_(torch.from_numpy(a))
torch.cuda.synchronize()
res["pageable_s"] = time.perf_counter() - t
cr = torch.cuda.cudart()
t = time.perf_counter()
rc = cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
t_reg = time.perf_counter() - t
t = time.perf_counter()
dev.copy_(torch.from_numpy(a), non_blocking=True)
torch.cuda.synchronize()
t_copy = time.perf_counter() - t
t = time.perf_counter()
cr.cudaHostUnregister(a.ctypes.data)
t_unreg = time.perf_counter() - t
res.update(register_rc=int(rc), register_s=t_reg, registered_copy_s=t_copy, unregister_s=t_unreg)
# staging ring: host threads memcpy chunks into pinned buffers, DMA overlapped
chunk = 16 << 20  # elements per chunk (128 MB)
ring = [torch.empty(chunk, dtype=torch.float64).pin_memory() for _ in range(4)]
evs = [None] * 4
s = torch.cuda.Stream()
src = torch.from_numpy(a)
pool = ThreadPoolExecutor(8)


def fill(buf, lo, hi):
    n = hi - lo
    parts = 8
    step = (n + parts - 1) // parts
    futs = [pool.submit(lambda i: buf[i * step:min(n, (i + 1) * step)].copy_(src[lo + i * step:min(hi, lo + (i + 1) * step)]), i)
            for i in range(parts) if i * step < n]
    for f in futs:
        f.result()


torch.cuda.synchronize()
t = time.perf_counter()
for k, lo in enumerate(range(0, D, chunk)):
    hi = min(D, lo + chunk)
    slot = k % 4
    if evs[slot] is not None:
        evs[slot].synchronize()
    fill(ring[slot], lo, hi)
    with torch.cuda.stream(s):
        dev[lo:hi].copy_(ring[slot][: hi - lo], non_blocking=True)
        evs[slot] = torch.cuda.Event()
        evs[slot].record(s)
torch.cuda.synchronize()
res["staged_ring_8threads_s"] = time.perf_counter() - t
res["gb"] = a.nbytes / 1e9
print(json.dumps(res))
