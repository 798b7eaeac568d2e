"""Multi-process helpers for the distributed tests (gloo on CPU, NCCL on GPUs)."""

from __future__ import annotations

import os
import socket

import numpy as np
import torch


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def init(rank: int, world: int, port: int, backend: str):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if backend == "nccl":
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)


def oracle_clip(grad, out, segments, limit, post_scale=1.0, norms=None, coefs=None, nonfinite=None):
    """CPU stand-in with BucketClipper.clip_cast's signature (test infrastructure, oracle arithmetic)."""
    from oracle import ddp_oracle as O

    for i, (a, o, n) in enumerate(segments):
        g = grad[a:a + n].double().numpy()
        out[o:o + n] = torch.from_numpy(O.clip_by_norm(g, limit) * post_scale).to(out.dtype)
        if norms is not None:
            norms[i] = float(np.linalg.norm(g))


def worker_grad(rank: int, dim: int) -> torch.Tensor:
    rng = np.random.default_rng(1000 + rank)
    g = rng.normal(size=dim) * (0.01 if rank % 2 == 0 else 0.3)
    return torch.tensor(g.astype(np.float32))
