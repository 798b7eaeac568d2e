"""The drop-in call end to end: sync_bucketwise(GradientState(numpy fp64 (1, D)), ClipConfig) -> numpy,
BERT-large D.  Times the constructor (staged H2D + finiteness pass) and the sync (K1 + D2H) apart.

    B2_STAGE_THREADS=N python tools/dropin_probe.py
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2402_02447_b200 as B  # noqa: E402
from paper_2402_02447_b200 import synthetic  # noqa: E402

D = synthetic.BERT_LARGE_DIM
w = (np.random.default_rng(0).standard_normal((1, D)) * 1e-3)
layout = B.equal_bucket_layout(D, 52)
cfg = B.ClipConfig(1.0, "bucket_wise")
ts = []
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = B.GradientState(w, layout)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    out = B.sync_bucketwise(st, cfg)
    t2 = time.perf_counter()
    del st, out
    ts.append((t1 - t0, t2 - t1))
ctor, sync = (float(np.median([t[i] for t in ts[1:]])) for i in (0, 1))
print(json.dumps({"threads": int(os.environ.get("B2_STAGE_THREADS", "8")), "ctor_ms": ctor * 1e3, "sync_ms": sync * 1e3,
                  "gbs": 2 * w.nbytes / (ctor + sync) / 1e9}))
