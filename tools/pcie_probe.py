"""PCIe floor of the e2e step: 1.34 GB pinned H2D alone, D2H alone, and both at once."""
import json
import time

import torch

n = 335_141_888
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float32, device="cuda")
d_b = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


th = t(lambda: d_a.copy_(h_in, non_blocking=True))
td = t(lambda: h_out.copy_(d_b, non_blocking=True))
tb = t(both)
gb = n * 4 / 1e9
print(json.dumps({"bytes": n * 4, "h2d_gbs": gb / th, "d2h_gbs": gb / td, "both_ms": tb * 1e3,
                  "both_gbs_per_dir": gb / tb, "e2e_floor_n1_gbs": gb / tb}))
