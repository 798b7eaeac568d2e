"""H1 across ranks: per-bucket fused clip on the compute stream, NCCL allreduce on a side stream.

One process per GPU (torch.distributed, backend "nccl").  Rank r holds worker
row r of the reference's (K, D) matrix (gradsync.py:43-48); the clip needs no
collective (it is purely local — the point of clipping *before* allreduce,
paper Algorithm 1), and each bucket is then averaged with
one allreduce, in reverse bucket order (gradsync.py:157), on a comm stream
event-chained after that bucket's K1 launch so the transfer of bucket b
overlaps the clip (and, in training, the backward) of bucket b-1.

``BucketwiseSync``   — owns the clipper, the comm stream and the comm buffer;
                       ``launch_bucket(b)`` / ``sync(grad)`` enqueue without
                       host synchronisation.
``bucketwise_clip_hook`` — a ``DistributedDataParallel`` communication hook
                       with the same semantics for DDP's own buckets.
"""

from __future__ import annotations

import math
from typing import Sequence

import torch
import torch.distributed as dist

from .gradsync import BucketClipper, ClipConfig, ClipMode


def _avg_op(group) -> tuple:
    """(op, post_scale): NCCL has a native average; gloo sums and K1 folds in 1/K."""
    backend = dist.get_backend(group)
    if backend == "nccl":
        return dist.ReduceOp.AVG, 1.0
    return dist.ReduceOp.SUM, 1.0 / dist.get_world_size(group)


class BucketwiseSync:
    """Bucket-wise clip-before-allreduce of one flat gradient vector per rank.

    ``layout`` is the contiguous bucket partition of the flat gradient
    (``capped_bucket_layout`` gives DDP's 25 MiB buckets).  The comm buffer
    dtype is bf16 (throughput) or fp32 (parity).  ``clip`` may be replaced by
    any callable with BucketClipper.clip_cast's signature (the CPU tests inject
    the oracle there to exercise the multi-rank orchestration under gloo).
    """

    def __init__(self, layout: Sequence, cfg: ClipConfig, comm_dtype=torch.bfloat16, group=None,
                 device=None, clip=None, ctas_per_sm: int = 0):
        if ClipConfig(cfg.threshold, cfg.mode).mode is not ClipMode.BUCKET_WISE:
            raise ValueError(f"config mode is {cfg.mode.value}, expected {ClipMode.BUCKET_WISE.value}")
        self.layout = tuple((int(a), int(b)) for a, b in layout)
        self.limit = cfg.threshold / math.sqrt(len(self.layout))  # gradsync.py:155
        self.group = group
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        self.dim = self.layout[-1][1]
        self.comm = torch.empty(self.dim, dtype=comm_dtype, device=self.device)
        self.op, self.post_scale = _avg_op(group)
        self.is_cuda = self.device.type == "cuda"
        if self.is_cuda:
            self.compute = torch.cuda.current_stream(self.device)
            self.side = torch.cuda.Stream(device=self.device)
            self.events = [torch.cuda.Event() for _ in self.layout]
        self.clip = clip if clip is not None else BucketClipper(device=self.device, ctas_per_sm=ctas_per_sm).clip_cast
        self.norms = torch.zeros(len(self.layout), dtype=torch.float64, device=self.device)
        self.works: list = []

    def launch_bucket(self, grad: torch.Tensor, b: int) -> None:
        """K1 for bucket b on the compute stream, then its allreduce on the side stream."""
        a, e = self.layout[b]
        self.clip(grad, self.comm, [(a, a, e - a)], self.limit, self.post_scale, self.norms[b:b + 1])
        if self.is_cuda:
            ev = self.events[b]
            ev.record(self.compute)
            self.side.wait_event(ev)
            with torch.cuda.stream(self.side):
                self.works.append(dist.all_reduce(self.comm[a:e], op=self.op, group=self.group, async_op=True))
        else:
            self.works.append(dist.all_reduce(self.comm[a:e], op=self.op, group=self.group, async_op=True))

    def sync(self, grad: torch.Tensor) -> torch.Tensor:
        """All buckets in backward order; returns the averaged comm buffer (not yet waited)."""
        if grad.numel() != self.dim:
            raise ValueError(f"gradient has {grad.numel()} elements, layout covers {self.dim}")
        for b in reversed(range(len(self.layout))):
            self.launch_bucket(grad, b)
        return self.comm

    def wait(self) -> torch.Tensor:
        """Join the side stream into the current stream (no host block for NCCL)."""
        for w in self.works:
            w.wait()
        self.works.clear()
        if self.is_cuda:
            torch.cuda.current_stream(self.device).wait_stream(self.side)
        return self.comm


class _HookState:
    def __init__(self, cfg: ClipConfig, num_buckets: int, process_group=None):
        self.limit = cfg.threshold / math.sqrt(num_buckets)
        self.group = process_group
        self.clipper = None
        self.norms = {}


def bucketwise_clip_hook(state: _HookState, bucket):
    """DDP comm hook: fused clip (K1) of the bucket at c/sqrt(B), then NCCL average.

    Register with ``model.register_comm_hook(make_hook_state(cfg, B), bucketwise_clip_hook)``.
    B must be fixed up front (use static_graph or a layout computed from the
    parameter sizes), because the threshold is c/sqrt(B) (gradsync.py:155).
    """
    buf = bucket.buffer()
    if state.clipper is None:
        state.clipper = BucketClipper(device=buf.device)
    op, post = _avg_op(state.group)
    n = buf.numel()
    norm = torch.empty(1, dtype=torch.float64, device=buf.device)
    state.clipper.clip_cast(buf, buf, [(0, 0, n)], state.limit, post, norms=norm)  # in place
    state.norms[bucket.index()] = norm
    fut = dist.all_reduce(buf, op=op, group=state.group, async_op=True).get_future()
    return fut.then(lambda f: f.value()[0])


def make_hook_state(cfg: ClipConfig, num_buckets: int, process_group=None) -> _HookState:
    if ClipConfig(cfg.threshold, cfg.mode).mode is not ClipMode.BUCKET_WISE:
        raise ValueError(f"config mode is {cfg.mode.value}, expected {ClipMode.BUCKET_WISE.value}")
    return _HookState(cfg, num_buckets, process_group)
