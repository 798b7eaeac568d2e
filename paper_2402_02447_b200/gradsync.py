"""H1 — bucket-wise gradient clipping before allreduce, on B200.

Drop-in for the reference module ``ddpsim.gradsync`` (gradsync.py:1-191): the
same names, arguments, modes and ``ValueError`` messages, but every pass over
gradient data runs in the sm_100a kernels of ``_native/libb2ddp.so``:

* K1 ``b2_bucket_clip_cast`` — per-bucket norm + clip coefficient + scale/cast
  (clip_by_norm, gradsync.py:106-116, per worker and bucket as in :157-160);
* K1b ``b2_weighted_mean`` — the K-worker pairwise-tree mean
  (allreduce_mean, :119-128) for the single-process K>1 state.

Array-like inputs (numpy, lists) are uploaded and results come back as fp64
numpy arrays, like the reference.  CUDA tensors stay on the device (fp32 or
fp64) and results are CUDA tensors.  ``BucketClipper`` is the low-level entry
the DDP hook and the benchmark use (fp32 gradients -> bf16/fp32 comm buffer,
no host synchronisation).
"""

from __future__ import annotations

import math
import os
import threading
from dataclasses import dataclass
from enum import Enum
from typing import Any, Sequence

import numpy as np
import torch

from . import _lib

BERT_BUCKET_ELEMS = 25 * 1024 * 1024 // 4  # 25 MiB of fp32 = 6,553,600 elements


class ClipMode(str, Enum):
    AFTER_ALLREDUCE = "after_allreduce"
    BEFORE_ALLREDUCE = "before_allreduce"
    BUCKET_WISE = "bucket_wise"


def equal_bucket_layout(dim: int, num_buckets: int) -> tuple:
    """Contiguous equal ranges over [0, dim); the last one takes the remainder."""
    if num_buckets < 1:
        raise ValueError(f"num_buckets must be >= 1, got {num_buckets}")
    if dim < num_buckets:
        raise ValueError(f"cannot split dimension {dim} into {num_buckets} buckets")
    step = dim // num_buckets
    edges = [k * step for k in range(num_buckets)] + [dim]
    return tuple((edges[k], edges[k + 1]) for k in range(num_buckets))


def capped_bucket_layout(dim: int, bucket_elems: int = BERT_BUCKET_ELEMS) -> tuple:
    """Fixed-capacity buckets (DDP-style 25 MiB fp32), the last one smaller."""
    if dim < 1 or bucket_elems < 1:
        raise ValueError("dim and bucket_elems must be >= 1")
    return tuple((a, min(a + bucket_elems, dim)) for a in range(0, dim, bucket_elems))


_STAGE_ELEMS = 8 << 20  # elements per pinned staging slot (64 MB of fp64; 32 MB slots measured 10 % slower)
_STAGE_SLOTS = 4
_STAGE_THREADS = int(os.environ.get("B2_STAGE_THREADS", "8"))  # host threads filling a slot
_staging: dict = {}
_staging_lock = threading.Lock()  # one ring per (dtype, device); callers on several threads take turns


def _staged_h2d(src: torch.Tensor) -> torch.Tensor:
    """Host (pageable) -> device through a ring of pinned slots filled by host threads.

    A caller's numpy array is pageable: one plain copy runs at ~11 GB/s on the
    GPU box, while 8 threads filling pinned slots (torch copies release the
    GIL) overlap with the DMA of the previous slot: ~35 GB/s for the 2.68 GB
    fp64 BERT-large state (tools/pinning_probe.py).  Small inputs copy directly.
    """
    flat = src.reshape(-1)
    n = flat.numel()
    out = torch.empty(src.shape, dtype=src.dtype, device="cuda")
    if n * flat.element_size() < (64 << 20):
        out.copy_(src)
        return out
    key = (src.dtype, torch.cuda.current_device())
    with _staging_lock:
        return _staged_h2d_locked(flat, out, key, src.dtype)


def _staged_h2d_locked(flat: torch.Tensor, out: torch.Tensor, key, dtype) -> torch.Tensor:
    from concurrent.futures import ThreadPoolExecutor

    n = flat.numel()
    st = _staging.get(key)
    if st is None:
        st = _staging[key] = {
            "slots": [torch.empty(_STAGE_ELEMS, dtype=dtype).pin_memory() for _ in range(_STAGE_SLOTS)],
            "events": [None] * _STAGE_SLOTS, "stream": torch.cuda.Stream(),
            "pool": ThreadPoolExecutor(max_workers=_STAGE_THREADS)}
    slots, evs, stream, pool = st["slots"], st["events"], st["stream"], st["pool"]
    dst = out.reshape(-1)
    stream.wait_stream(torch.cuda.current_stream())
    for k, lo in enumerate(range(0, n, _STAGE_ELEMS)):
        hi = min(n, lo + _STAGE_ELEMS)
        i = k % _STAGE_SLOTS
        if evs[i] is not None:
            evs[i].synchronize()  # the slot's previous DMA has drained
        buf, m = slots[i], hi - lo
        step = (m + _STAGE_THREADS - 1) // _STAGE_THREADS
        futs = [pool.submit(buf[a:min(m, a + step)].copy_, flat[lo + a:lo + min(m, a + step)])
                for a in range(0, m, step)]
        for f in futs:
            f.result()
        with torch.cuda.stream(stream):
            dst[lo:hi].copy_(buf[:m], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            evs[i] = ev
    torch.cuda.current_stream().wait_stream(stream)
    out.record_stream(stream)
    return out


def _to_device_matrix(workers) -> tuple[torch.Tensor, bool]:
    """(K, D) CUDA tensor + whether the caller handed us host data."""
    if isinstance(workers, torch.Tensor):
        host = not workers.is_cuda
        t = workers
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
    else:
        host = True
        try:
            arr = np.asarray(workers, dtype=float)
        except ValueError:
            raise ValueError("workers have mismatched dimensions") from None
        t = torch.from_numpy(np.ascontiguousarray(arr))
    if t.ndim != 2 or t.shape[0] < 1 or t.shape[1] < 1:
        raise ValueError(f"expected a (workers, dim) matrix, got shape {tuple(t.shape)}")
    _lib.load()
    if t.is_cuda:
        t = t.contiguous()
    elif t.is_pinned():
        t = t.contiguous().to("cuda", non_blocking=True)
    else:
        t = _staged_h2d(t.contiguous())
    return t, host


def _finite_or_raise(t: torch.Tensor, what: str) -> None:
    """Reject inf/nan (gradsync.py:189-190) with one K1 norm pass (its non-finite flags)."""
    m = t.reshape(t.shape[0], -1) if t.ndim > 1 else t.reshape(1, -1)
    K, D = m.shape
    flags = torch.empty(K, dtype=torch.int32, device=m.device)
    _clipper().clip_cast(m, None, [(k * m.stride(0), 0, D) for k in range(K)], 1.0, nonfinite=flags)
    if bool(flags.any()):
        raise ValueError(f"{what} has non-finite components")


@dataclass
class GradientState:
    """K per-worker flat gradients (rows of a CUDA matrix) + a bucket partition."""

    workers: Any
    bucket_layout: tuple

    def __post_init__(self):
        self.workers, self._host = _to_device_matrix(self.workers)
        _finite_or_raise(self.workers, "gradient state")
        layout = tuple((int(a), int(b)) for a, b in self.bucket_layout)
        self.bucket_layout = layout
        dim = self.workers.shape[1]
        if not layout:
            raise ValueError("bucket_layout must have at least one bucket")
        edge = 0
        for a, b in layout:
            if a != edge or b <= a:
                raise ValueError(
                    f"bucket_layout must be disjoint contiguous ranges covering [0, {dim}), got {layout}"
                )
            edge = b
        if edge != dim:
            raise ValueError(f"bucket_layout covers [0, {edge}), expected [0, {dim})")

    @property
    def num_workers(self) -> int:
        return self.workers.shape[0]

    @property
    def dim(self) -> int:
        return self.workers.shape[1]

    @property
    def num_buckets(self) -> int:
        return len(self.bucket_layout)


def gradient_state_from_dict(doc: dict) -> GradientState:
    """Build a state from a plain document (gradsync.py:81-92)."""
    workers, _ = _to_device_matrix(doc["workers"])
    if "bucket_layout" in doc:
        layout = tuple((int(a), int(b)) for a, b in doc["bucket_layout"])
    else:
        layout = equal_bucket_layout(workers.shape[1], int(doc.get("num_buckets", 1)))
    state = GradientState(workers, layout)
    state._host = not isinstance(doc["workers"], torch.Tensor) or not doc["workers"].is_cuda
    return state


@dataclass(frozen=True)
class ClipConfig:
    threshold: float
    mode: ClipMode

    def __post_init__(self):
        object.__setattr__(self, "mode", ClipMode(self.mode))
        if not (self.threshold > 0 and math.isfinite(self.threshold)):
            raise ValueError(f"threshold must be positive and finite, got {self.threshold}")


# ---------------------------------------------------------------------------
# low-level launcher (the hot path)

_DT = {torch.float32: _lib.B2_F32, torch.bfloat16: _lib.B2_BF16, torch.float64: _lib.B2_F64}


class BucketClipper:
    """Launches K1 on one stream with its own zeroed workspace.

    ``clip_cast(grad, out, segments, limit)`` enqueues one cooperative kernel
    for all given segments (≤128 per launch); nothing synchronises the host.
    ``segments`` is a sequence of (in_offset, out_offset, length).
    """

    def __init__(self, device=None, stream: torch.cuda.Stream | None = None, ctas_per_sm: int = 0):
        self.lib = _lib.load()
        self.device = torch.device(device if device is not None else "cuda")
        self.stream = stream
        self.ctas_per_sm = int(ctas_per_sm)
        nbytes = self.lib.b2_clip_workspace_bytes()
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        _lib.check(self.lib.b2_clip_workspace_init(self.workspace.data_ptr(), nbytes, self._sp()))

    def _sp(self) -> int:
        return _lib.stream_ptr(self.stream)

    def clip_cast(self, grad: torch.Tensor, out: torch.Tensor | None, segments: Sequence,
                  limit: float, post_scale: float = 1.0, norms: torch.Tensor | None = None,
                  coefs: torch.Tensor | None = None, nonfinite: torch.Tensor | None = None) -> None:
        self.prepare(grad, out, segments, limit, post_scale, norms, coefs, nonfinite)()

    def prepare(self, grad: torch.Tensor, out: torch.Tensor | None, segments: Sequence,
                limit: float, post_scale: float = 1.0, norms: torch.Tensor | None = None,
                coefs: torch.Tensor | None = None, nonfinite: torch.Tensor | None = None):
        """Validate once and return a zero-argument launcher (per-bucket hot loops, graph capture)."""
        segs = list(segments)
        if grad.dtype not in (torch.float32, torch.float64) or not grad.is_cuda:
            raise ValueError("grad must be a CUDA float32/float64 tensor")
        if out is not None and (out.dtype not in _DT or not out.is_cuda):
            raise ValueError("out must be a CUDA float32/bfloat16/float64 tensor")
        n_in = grad.numel()
        for a, o, n in segs:
            if a < 0 or n < 0 or a + n > n_in or (out is not None and (o < 0 or o + n > out.numel())):
                raise ValueError(f"segment ({a}, {o}, {n}) is out of bounds")
        for t in (norms, coefs):
            if t is not None and (t.dtype != torch.float64 or t.numel() < len(segs)):
                raise ValueError("norms/coefs must be float64 tensors with one entry per segment")
        if nonfinite is not None and (nonfinite.dtype != torch.int32 or nonfinite.numel() < len(segs)):
            raise ValueError("nonfinite must be an int32 tensor with one entry per segment")
        ins = _lib.i64_array(s[0] for s in segs)
        outs = _lib.i64_array(s[1] for s in segs)
        lens = _lib.i64_array(s[2] for s in segs)
        ws = self.workspace
        fn = self.lib.b2_bucket_clip_cast
        args = (
            grad.data_ptr(), _DT[grad.dtype],
            out.data_ptr() if out is not None else None, _DT[out.dtype] if out is not None else 0,
            ins, outs, lens, len(segs), float(limit), float(post_scale),
            norms.data_ptr() if norms is not None else None,
            coefs.data_ptr() if coefs is not None else None,
            nonfinite.data_ptr() if nonfinite is not None else None,
            ws.data_ptr(), ws.numel(), self.ctas_per_sm, self._sp(),
        )
        keep = (grad, out, norms, coefs, nonfinite, ws)  # tensors must outlive the launcher
        check = _lib.check

        def launch():
            check(fn(*args))
            return keep

        return launch

    def weighted_mean(self, mat: torch.Tensor, coefs: torch.Tensor, bounds: Sequence[int],
                      out: torch.Tensor) -> None:
        K, D = mat.shape
        b = _lib.i64_array(bounds)
        rc = self.lib.b2_weighted_mean(
            mat.data_ptr(), _DT[mat.dtype], K, D, mat.stride(0), coefs.data_ptr(), b,
            len(bounds) - 1, out.data_ptr(), _DT[out.dtype], self._sp(),
        )
        _lib.check(rc)


_clippers: dict = {}


def _clipper() -> BucketClipper:
    """One clipper (workspace) per (device, current stream)."""
    s = torch.cuda.current_stream()
    key = (s.device.index, int(s.cuda_stream))
    c = _clippers.get(key)
    if c is None:
        c = _clippers[key] = BucketClipper(device=s.device, stream=s)
    return c


def _result(t: torch.Tensor, host: bool):
    """Host callers get numpy; the D2H lands in (cached) pinned memory at full PCIe rate."""
    if not host:
        return t
    dst = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    dst.copy_(t)
    return dst.numpy()


def _raise_if_flagged(flags: torch.Tensor) -> None:
    if bool(flags.any()):
        raise ValueError("gradient has non-finite components")


# ---------------------------------------------------------------------------
# reference API


def clip_by_norm(g, limit: float):
    """Rescale g to L2 norm ``limit`` iff its norm reaches the limit (gradsync.py:106-116)."""
    if limit <= 0:
        raise ValueError(f"limit must be > 0, got {limit}")
    arr = None
    if isinstance(g, torch.Tensor):
        host = not g.is_cuda
        v = g if g.dtype in (torch.float32, torch.float64) else g.to(torch.float64)
    else:
        host = True
        arr = np.asarray(g, dtype=float)  # a float64 ndarray comes back as itself (:110)
        v = torch.from_numpy(np.ascontiguousarray(arr))
    src = v
    v = v.reshape(-1).to("cuda").contiguous()
    c = _clipper()
    norms = torch.empty(1, dtype=torch.float64, device=v.device)
    flags = torch.empty(1, dtype=torch.int32, device=v.device)
    out = torch.empty_like(v)
    c.clip_cast(v, out, [(0, 0, v.numel())], limit, norms=norms, nonfinite=flags)
    _raise_if_flagged(flags)
    if float(norms.item()) >= limit:
        return _result(out.reshape(src.shape), host)
    if arr is not None:
        return arr  # unchanged: the same array object (:116)
    return src.numpy() if host else src


def allreduce_mean(workers):
    """Elementwise mean over workers with the reference's pairwise tree (:119-128)."""
    mat, host = _to_device_matrix(workers)
    _finite_or_raise(mat, "gradient state")
    out = torch.empty(mat.shape[1], dtype=mat.dtype, device=mat.device)
    ones = torch.ones(mat.shape[0], dtype=torch.float64, device=mat.device)
    _clipper().weighted_mean(mat, ones, [0, mat.shape[1]], out)
    return _result(out, host)


def _require_mode(cfg: ClipConfig, expected: ClipMode) -> None:
    if cfg.mode is not expected:
        raise ValueError(f"config mode is {cfg.mode.value}, expected {expected.value}")


def sync_after(state: GradientState, cfg: ClipConfig):
    """Mean of the full vectors, then clip the mean to c (:131-134)."""
    _require_mode(cfg, ClipMode.AFTER_ALLREDUCE)
    W = state.workers
    c = _clipper()
    mean = torch.empty(W.shape[1], dtype=W.dtype, device=W.device)
    ones = torch.ones(W.shape[0], dtype=torch.float64, device=W.device)
    c.weighted_mean(W, ones, [0, W.shape[1]], mean)
    norms = torch.empty(1, dtype=torch.float64, device=W.device)
    flags = torch.empty(1, dtype=torch.int32, device=W.device)
    out = torch.empty_like(mean)
    c.clip_cast(mean, out, [(0, 0, mean.numel())], cfg.threshold, norms=norms, nonfinite=flags)
    _raise_if_flagged(flags)
    return _result(out if float(norms.item()) >= cfg.threshold else mean, state._host)


def sync_before(state: GradientState, cfg: ClipConfig):
    """Clip every worker's full vector to c, then the pairwise mean (:137-145)."""
    _require_mode(cfg, ClipMode.BEFORE_ALLREDUCE)
    return _clip_then_mean(state, ((0, state.dim),), cfg.threshold)


def sync_bucketwise(state: GradientState, cfg: ClipConfig):
    """Clip each worker's bucket to c/sqrt(B), then average bucket by bucket (:148-162)."""
    _require_mode(cfg, ClipMode.BUCKET_WISE)
    limit = cfg.threshold / math.sqrt(state.num_buckets)
    return _clip_then_mean(state, state.bucket_layout, limit)


def _clip_then_mean(state: GradientState, layout, limit: float):
    W = state.workers
    K, D = W.shape
    B = len(layout)
    c = _clipper()
    out = torch.empty(D, dtype=W.dtype, device=W.device)
    flags = torch.empty(K * B, dtype=torch.int32, device=W.device)
    if K == 1:
        # one fused pass: norm + coef + scale straight into the result;
        # buckets walked in reverse like a backward pass (:157)
        segs = [(a, a, b - a) for a, b in reversed(layout)]
        c.clip_cast(W, out, segs, limit, nonfinite=flags)
    else:
        coefs = torch.empty(K * B, dtype=torch.float64, device=W.device)
        ld = W.stride(0)
        segs = [(k * ld + a, 0, b - a) for k in range(K) for a, b in layout]
        c.clip_cast(W, None, segs, limit, coefs=coefs, nonfinite=flags)
        c.weighted_mean(W, coefs, [layout[0][0]] + [b for _, b in layout], out)
    _raise_if_flagged(flags)
    return _result(out, state._host)


def _check_layout(layout, dim: int) -> tuple:
    layout = tuple((int(a), int(b)) for a, b in layout)
    if not layout:
        raise ValueError("bucket_layout must have at least one bucket")
    edge = 0
    for a, b in layout:
        if a != edge or b <= a:
            raise ValueError(f"bucket_layout must be disjoint contiguous ranges covering [0, {dim}), got {layout}")
        edge = b
    if edge != dim:
        raise ValueError(f"bucket_layout covers [0, {edge}), expected [0, {dim})")
    return layout


def sync_bucketwise_host(workers, bucket_layout, cfg: ClipConfig, out: torch.Tensor | None = None):
    """Host-resident fast path of ``sync_bucketwise(GradientState(workers, layout), cfg)``.

    Same validation, errors and result as the two reference calls
    (gradsync.py:43-78, 148-162), but streamed bucket by bucket in the
    reference's reverse order over three CUDA streams — host->device copy of
    bucket b, K1 clip of b (with its non-finite flag), device->host copy of
    b — so both PCIe directions run at once instead of one after the other.
    A non-finite input raises ``ValueError`` ("gradient state has non-finite
    components") before any result is returned.  ``out`` may be a pinned
    host tensor to receive the result (else a pinned one is allocated): of
    the input's dtype (the result comes back as numpy), or bfloat16 — the
    comm-buffer dtype of the multi-rank step — which halves the device->host
    bytes and comes back as that torch tensor.  The host input should be
    pinned for full PCIe rate.  Single worker (K = 1); K > 1 goes through
    GradientState + sync_bucketwise.
    """
    _require_mode(cfg, ClipMode.BUCKET_WISE)
    src = workers if isinstance(workers, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(workers, dtype=float)))
    if src.ndim != 2 or src.shape[0] < 1 or src.shape[1] < 1:
        raise ValueError(f"expected a (workers, dim) matrix, got shape {tuple(src.shape)}")
    if src.is_cuda or src.shape[0] != 1:
        return sync_bucketwise(GradientState(workers, bucket_layout), cfg)
    if src.dtype not in (torch.float32, torch.float64):
        src = src.to(torch.float64)
    _lib.load()
    D = src.shape[1]
    layout = _check_layout(bucket_layout, D)
    limit = cfg.threshold / math.sqrt(len(layout))
    g = src.reshape(-1)
    if not g.is_contiguous():
        g = g.contiguous()
    dev = torch.device("cuda", torch.cuda.current_device())
    compute = torch.cuda.current_stream(dev)
    h2d, d2h = _host_streams(dev)
    d_in = torch.empty(D, dtype=g.dtype, device=dev)
    if out is None:
        out = torch.empty(D, dtype=g.dtype, pin_memory=True)
    elif out.numel() != D or out.dtype not in (g.dtype, torch.bfloat16) or out.is_cuda:
        raise ValueError(f"out must be a host {g.dtype} or bfloat16 tensor of {D} elements")
    d_out = torch.empty(D, dtype=out.dtype, device=dev)
    flags = torch.empty(len(layout), dtype=torch.int32, device=dev)
    c = _clipper()
    h2d.wait_stream(compute)  # d_in / d_out are fresh allocations of the compute stream
    for j, (a, b) in enumerate(reversed(layout)):  # bucket B first (:157)
        with torch.cuda.stream(h2d):
            d_in[a:b].copy_(g[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(h2d)
        compute.wait_event(ev)
        c.clip_cast(d_in, d_out, [(a, a, b - a)], limit, nonfinite=flags[j:j + 1])
        ev2 = torch.cuda.Event()
        ev2.record(compute)
        d2h.wait_event(ev2)
        with torch.cuda.stream(d2h):
            out[a:b].copy_(d_out[a:b], non_blocking=True)
    compute.wait_stream(d2h)
    d_in.record_stream(h2d)
    d_out.record_stream(d2h)
    if bool(flags.any()):  # synchronises: every copy has landed
        raise ValueError("gradient state has non-finite components")
    return out if out.dtype == torch.bfloat16 else out.numpy()


_host_stream_cache: dict = {}


def _host_streams(dev):
    s = _host_stream_cache.get(dev.index)
    if s is None:
        s = _host_stream_cache[dev.index] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    return s


_SYNC_FNS = {
    ClipMode.AFTER_ALLREDUCE: sync_after,
    ClipMode.BEFORE_ALLREDUCE: sync_before,
    ClipMode.BUCKET_WISE: sync_bucketwise,
}


def synchronize(state: GradientState, cfg: ClipConfig):
    """Dispatch on cfg.mode (:165-174)."""
    return _SYNC_FNS[cfg.mode](state, cfg)
