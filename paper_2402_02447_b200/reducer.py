"""Algorithm 1 as a gradient reducer: bucket-wise clip before allreduce, overlapped with backward.

Paper Algorithm 1 / sync_bucketwise (gradsync.py:148-162)
applied to a real model's gradients, without DistributedDataParallel:

* every trainable parameter's ``.grad`` is a view into ONE flat fp32 buffer
  laid out in parameter order, cut into contiguous buckets of at most
  ``bucket_cap_mb`` up front, walking the parameters in reverse (backward)
  order like DDP.  B — and with it the threshold c/sqrt(B) (gradsync.py:155)
  — is therefore known before iteration 0 (DDP only knows its buckets after
  it has rebuilt them at iteration 1);
* a post-accumulate-grad hook counts each bucket's parameters; when the last
  one lands, K1 clips the bucket at c/sqrt(B) and casts it into the comm
  buffer (bf16 by default) on the compute stream, the comm stream averages it
  with ncclAllReduce, and casts the average back into the fp32 gradients —
  all while backward continues with the earlier layers;
* ``finish()`` fires buckets that received no gradient (unused parameters),
  joins the comm stream into the compute stream and raises the reference's
  ValueError if any rank's gradient held inf/nan.

Buckets are fired in reverse layout order as backward produces them, which
is the order sync_bucketwise walks them; the result does not depend on the
order (each bucket's clip is local, gradsync.py:150-151).
"""

from __future__ import annotations

import math
from typing import Iterable

import torch
import torch.distributed as dist

from .gradsync import BucketClipper, ClipConfig, ClipMode


class BucketwiseReducer:
    def __init__(self, params: Iterable[torch.nn.Parameter], cfg: ClipConfig, bucket_cap_mb: float = 25.0,
                 comm_dtype: torch.dtype = torch.bfloat16, group=None, device=None):
        cfg = ClipConfig(cfg.threshold, cfg.mode)
        if cfg.mode is not ClipMode.BUCKET_WISE:
            raise ValueError(f"config mode is {cfg.mode.value}, expected {ClipMode.BUCKET_WISE.value}")
        self.params = [p for p in params if p.requires_grad]
        if not self.params:
            raise ValueError("no trainable parameters")
        self.device = torch.device(device) if device is not None else self.params[0].device
        if self.device.type != "cuda":
            raise ValueError("BucketwiseReducer runs on CUDA parameters")
        if any(p.dtype != torch.float32 for p in self.params):
            raise ValueError("BucketwiseReducer keeps fp32 gradients (fp32 master parameters)")
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        # flat fp32 gradient buffer in parameter order; .grad of every parameter is a view
        offs, o = [], 0
        for p in self.params:
            offs.append(o)
            o += p.numel()
        self.dim = o
        self.flat = torch.zeros(self.dim, dtype=torch.float32, device=self.device)
        for p, a in zip(self.params, offs):
            p.grad = self.flat[a:a + p.numel()].view_as(p)
        # buckets: walk the parameters backward, close a bucket once it reaches the cap
        cap = int(bucket_cap_mb * 1024 * 1024) // 4
        bounds, end, size = [], self.dim, 0
        for i in reversed(range(len(self.params))):
            size += self.params[i].numel()
            if size >= cap and i > 0:
                bounds.append(offs[i])
                size = 0
        edges = [0] + sorted(bounds) + [self.dim]
        self.layout = tuple((edges[k], edges[k + 1]) for k in range(len(edges) - 1))
        self.limit = cfg.threshold / math.sqrt(len(self.layout))  # c / sqrt(B), gradsync.py:155
        bucket_of = []
        for a in offs:
            b = 0
            while self.layout[b][1] <= a:
                b += 1
            bucket_of.append(b)
        self._bucket_of = bucket_of
        self._count = [0] * len(self.layout)
        for b in bucket_of:
            self._count[b] += 1
        self._pending = list(self._count)
        self.comm = torch.empty(self.dim, dtype=comm_dtype, device=self.device)
        self.compute = torch.cuda.current_stream(self.device)
        self.side = torch.cuda.Stream(device=self.device)
        self.events = [torch.cuda.Event() for _ in self.layout]
        self.clipper = BucketClipper(device=self.device)
        self.norms = torch.zeros(len(self.layout), dtype=torch.float64, device=self.device)
        self.nonfinite = torch.zeros(len(self.layout), dtype=torch.int32, device=self.device)
        self.nccl = None
        if self.world > 1:
            if dist.get_backend(group) != "nccl":
                raise ValueError("BucketwiseReducer averages over NCCL")
            from .ddp import NcclComm

            self.nccl = NcclComm(group)
        self.fired: list = []
        self._handles = [p.register_post_accumulate_grad_hook(self._make_hook(i)) for i, p in enumerate(self.params)]

    # ---------------------------------------------------------------- hooks
    def _make_hook(self, i: int):
        b = self._bucket_of[i]

        def hook(_p):
            self._pending[b] -= 1
            if self._pending[b] == 0:
                self._fire(b)
        return hook

    def _fire(self, b: int) -> None:
        a, e = self.layout[b]
        stream = torch.cuda.current_stream(self.device)  # backward's stream: K1 right behind the bucket's grads
        # K1: norm, coefficient c/sqrt(B)/norm (inclusive >=), scale + cast into the comm buffer
        self.clipper.clip_cast(self.flat, self.comm, [(a, a, e - a)], self.limit, 1.0, self.norms[b:b + 1],
                               nonfinite=self.nonfinite[b:b + 1])
        ev = self.events[b]
        ev.record(stream)
        self.side.wait_event(ev)
        if self.nccl is not None:
            self.nccl.all_reduce_avg(self.comm[a:e], stream=self.side)
        with torch.cuda.stream(self.side):
            self.flat[a:e].copy_(self.comm[a:e])  # the averaged bucket back into the fp32 gradients
        self.fired.append(b)

    # ---------------------------------------------------------------- step API
    def finish(self, check_finite: bool = True) -> None:
        """After backward: fire buckets nobody completed, join the comm stream, re-arm the counters."""
        for b in reversed(range(len(self.layout))):
            if self._pending[b] > 0:
                self._fire(b)
        torch.cuda.current_stream(self.device).wait_stream(self.side)
        self._pending = list(self._count)
        self.fired_order, self.fired = self.fired, []
        if check_finite:
            flags = self.nonfinite
            if self.world > 1:
                flags = flags.clone()
                dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=self.group)
            if bool(flags.any()):
                self.nonfinite.zero_()
                raise ValueError("gradient has non-finite components")

    def zero_grad(self) -> None:
        """Zero the gradients in place (keeps the .grad views into the flat buffer)."""
        self.flat.zero_()

    def remove(self) -> None:
        for h in self._handles:
            h.remove()
        self._handles = []
