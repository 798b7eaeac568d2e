"""H2 — presorted batch assignment, on B200 (drop-in for the presort half of ``ddpsim.balance``).

``assign_local_presort`` (balance.py:158-184) and ``assign_global_presort``
(:83-88) sort every pool by (-length, id) with a stable sort and deal it
raster/snake, all pools in one call: pools of <= 4096 samples with K3
``b2_presort_deal`` (one CTA per pool), larger pools — a global presort over a
whole batch, a whole rank shard — with K5 ``b2_presort_sort_deal`` (a
device-wide onesweep radix sort).  ``presort_deal`` is the tensor fast path
(int32 ids/lengths in HBM -> dealt ids + int64 token sums) used for whole
epochs of node-steps; ``sort_shard`` is the per-rank stable radix sort.

Out of scope (paper baselines, not the proposed path — SURVEY §2.1):
``assign_none``, ``pack_corpus``, ``assign_packing``.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .seqdata import Sample, Topology

MAX_POOL = 4096  # samples per pool one K3 CTA sorts; larger pools take the device-wide sort (K5)


class ScanPattern(str, Enum):
    RASTER = "raster"
    SNAKE = "snake"


@dataclass
class Assignment:
    """Per-GPU ordered samples + exact token totals (balance.py:40-51)."""

    per_gpu: list
    token_counts: tuple

    def to_dict(self) -> dict:
        return {
            "per_gpu_ids": [[s.id for s in gpu] for gpu in self.per_gpu],
            "token_counts": list(self.token_counts),
        }


def presort_deal(ids: torch.Tensor, lens: torch.Tensor, seg_len: int, lanes: int,
                 scan: ScanPattern | str = ScanPattern.SNAKE, max_len: int | None = None,
                 max_id: int | None = None, with_pos: bool = False, stream=None,
                 workspace: torch.Tensor | None = None):
    """Sort + deal ``ids.numel() // seg_len`` consecutive pools on the device.

    Returns (out_ids[nseg, lanes, rows] int32, tokens[nseg, lanes] int64,
    pos or None, bad[1] int64).  ``max_len``/``max_id`` bound the radix key
    (defaults: 2^31-1, i.e. full width; tight bounds mean fewer digit passes
    for large pools); out-of-range samples are reported through ``bad``.
    Pools larger than ``MAX_POOL`` use the device-wide sort, whose scratch is
    ``workspace`` (allocated here when not given; see ``presort_workspace_bytes``).
    """
    scan = ScanPattern(scan)
    lib = _lib.load()
    if seg_len % lanes:
        raise ValueError(f"{seg_len} items do not divide over {lanes} GPUs")
    if ids.dtype != torch.int32 or lens.dtype != torch.int32 or not ids.is_cuda or not lens.is_cuda:
        raise ValueError("ids and lens must be int32 CUDA tensors")
    n = ids.numel()
    if lens.numel() != n or (seg_len and n % seg_len):
        raise ValueError("ids/lens must hold a whole number of pools of seg_len samples")
    nseg = n // seg_len if seg_len else 0
    rows = seg_len // lanes
    dev = ids.device
    max_len = int(max_len if max_len is not None else 2**31 - 1)
    max_id = int(max_id if max_id is not None else 2**31 - 1)
    out = torch.empty((nseg, lanes, rows), dtype=torch.int32, device=dev)
    pos = torch.empty((nseg, lanes, rows), dtype=torch.int32, device=dev) if with_pos else None
    tok = torch.empty((nseg, lanes), dtype=torch.int64, device=dev)
    bad = torch.empty(1, dtype=torch.int64, device=dev)
    scan_c = _lib.B2_SCAN_SNAKE if scan is ScanPattern.SNAKE else _lib.B2_SCAN_RASTER
    if seg_len <= MAX_POOL:
        rc = lib.b2_presort_deal(
            ids.data_ptr(), lens.data_ptr(), nseg, seg_len, lanes, scan_c, max_len, max_id,
            out.data_ptr(), pos.data_ptr() if pos is not None else None, tok.data_ptr(),
            bad.data_ptr(), _lib.stream_ptr(stream),
        )
    else:
        need = presort_workspace_bytes(nseg, seg_len, max_len, max_id, with_pos)
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(need, dtype=torch.uint8, device=dev)
        rc = lib.b2_presort_sort_deal(
            ids.data_ptr(), lens.data_ptr(), nseg, seg_len, lanes, scan_c, max_len, max_id,
            out.data_ptr(), pos.data_ptr() if pos is not None else None, tok.data_ptr(),
            bad.data_ptr(), workspace.data_ptr(), workspace.numel(), _lib.stream_ptr(stream),
        )
    _lib.check(rc)
    return (out, tok, pos, bad) if with_pos else (out, tok, None, bad)


def presort_workspace_bytes(nseg: int, seg_len: int, max_len: int, max_id: int, with_pos: bool = False) -> int:
    """Device scratch the device-wide sort (pools > MAX_POOL) needs; 0 for K3-sized pools."""
    if seg_len <= MAX_POOL:
        return 0
    need = int(_lib.load(require_device=False).b2_presort_workspace_bytes(nseg, seg_len, max_len, max_id,
                                                                          int(with_pos)))
    if need == 0:
        raise _lib.B2Error(f"no radix plan for pools of {seg_len} samples (max_len {max_len}, max_id {max_id})")
    return need


def sort_shard(ids: torch.Tensor, lens: torch.Tensor, max_len: int | None = None, max_id: int | None = None,
               with_pos: bool = False, stream=None):
    """The per-rank stable radix sort on length keys: one whole shard in (-length, id) order.

    This is _sorted_desc (balance.py:73-75) over a whole shard — K5 with one
    pool and one lane.  Returns (sorted ids int32, total tokens int64[1],
    input slots or None, bad[1]).
    """
    n = ids.numel()
    out, tok, pos, bad = presort_deal(ids, lens, n, 1, ScanPattern.RASTER, max_len, max_id, with_pos, stream)
    return out.reshape(-1), tok.reshape(-1), (pos.reshape(-1) if pos is not None else None), bad


def _deal_pools(pools: list, lanes: int, scan: ScanPattern) -> tuple:
    """K3 over equal-size host pools of Sample -> (per-lane Sample lists, tokens)."""
    seg_len = len(pools[0])
    if seg_len % lanes:
        raise ValueError(f"{seg_len} items do not divide over {lanes} GPUs")
    if seg_len == 0:
        return [[] for _ in range(lanes * len(pools))], tuple(0 for _ in range(lanes * len(pools)))
    flat = [s for pool in pools for s in pool]
    ids = np.fromiter((s.id for s in flat), dtype=np.int64, count=len(flat))
    lens = np.fromiter((s.length for s in flat), dtype=np.int64, count=len(flat))
    if ids.max() > 2**31 - 1 or lens.max() > 2**31 - 1:
        raise _lib.B2Error("sample ids and lengths must fit int32 on the device path")
    _lib.load()
    d_ids = torch.from_numpy(ids.astype(np.int32)).to("cuda", non_blocking=True)
    d_lens = torch.from_numpy(lens.astype(np.int32)).to("cuda", non_blocking=True)
    _, tok, pos, bad = presort_deal(d_ids, d_lens, seg_len, lanes, scan,
                                    max_len=int(lens.max()), max_id=int(ids.max()), with_pos=True)
    pos_h = pos.cpu().numpy().reshape(len(pools) * lanes, seg_len // lanes)
    per_gpu = [[flat[i] for i in row] for row in pos_h]
    return per_gpu, tuple(int(t) for t in tok.cpu().reshape(-1).tolist())


def assign_global_presort(batch: Sequence[Sample], topo: Topology,
                          scan: ScanPattern = ScanPattern.RASTER) -> Assignment:
    """Sort the whole batch (-length, id), deal across all GPUs (balance.py:83-88)."""
    scan = ScanPattern(scan)
    per_gpu, tok = _deal_pools([list(batch)], topo.total_gpus, scan)
    return Assignment(per_gpu=per_gpu, token_counts=tok)


def assign_local_presort(per_gpu_draws: Sequence[Sequence[Sample]], topo: Topology,
                         scan: ScanPattern = ScanPattern.SNAKE) -> Assignment:
    """Pool each node's GPU draws, sort (-length, id), deal among the node (balance.py:158-184)."""
    scan = ScanPattern(scan)
    if len(per_gpu_draws) != topo.total_gpus:
        raise ValueError(
            f"got draws for {len(per_gpu_draws)} GPUs, topology has {topo.total_gpus}"
        )
    sizes = {len(d) for d in per_gpu_draws}
    if len(sizes) > 1:
        raise ValueError(f"per-GPU draw counts differ: {sorted(sizes)}")
    g = topo.gpus_per_node
    pools = [
        [s for d in per_gpu_draws[node * g:(node + 1) * g] for s in d] for node in range(topo.num_nodes)
    ]
    per_gpu, tok = _deal_pools(pools, g, scan)
    return Assignment(per_gpu=per_gpu, token_counts=tok)
