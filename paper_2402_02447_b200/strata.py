"""H2 — length strata, on B200 (drop-in for ``ddpsim.strata``, strata.py:1-161).

* ``stratify`` / ``stratify_lengths`` run K2 ``b2_strata_partition`` (stratum
  histogram + stable partition) on the device.  ``stratify`` keeps the
  reference signature and returns ``Strata`` of ``Sample`` lists; the tensor
  form returns ``DeviceStrata`` (partitioned int32 ids + counts) and never
  leaves the GPU except for the ``nb`` stratum counts.
* ``allocate_counts`` is four floats of host arithmetic (strata.py:86-110) and
  stays on the host with the reference's exact numpy expression.
* ``draw_batch`` is the boundary input: draws come from numpy's PCG64
  ``Generator.choice`` (strata.py:113-161) and stay on the host so the draw
  sequence is bit-identical; a device port is SURVEY §8(f) row 2.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .seqdata import DEFAULT_BIN_BOUNDARIES, Sample

DEFAULT_STRATUM_BOUNDARIES = DEFAULT_BIN_BOUNDARIES
_I32_MAX = 2**31 - 1


@dataclass
class Strata:
    """Per-stratum sample pools (mutated by draw_batch) + probabilities."""

    boundaries: tuple
    buckets: list
    probs: tuple

    @property
    def num_strata(self) -> int:
        return len(self.boundaries)

    @property
    def remaining(self) -> int:
        return sum(len(pool) for pool in self.buckets)


@dataclass(frozen=True)
class StratumAllocation:
    counts: tuple
    local_batch: int

    def __post_init__(self):
        if any(c < 0 for c in self.counts):
            raise ValueError(f"counts must be non-negative, got {self.counts}")
        if sum(self.counts) != self.local_batch:
            raise ValueError(
                f"counts {self.counts} sum to {sum(self.counts)}, "
                f"expected local_batch {self.local_batch}"
            )


@dataclass
class DeviceStrata:
    """Stratified ids resident in HBM: ``ids[offsets[k]:offsets[k]+counts[k]]`` is stratum k."""

    boundaries: tuple
    ids: torch.Tensor
    counts: tuple
    probs: tuple

    @property
    def offsets(self) -> tuple:
        return tuple(int(x) for x in np.concatenate([[0], np.cumsum(self.counts)[:-1]]))

    def pool(self, k: int) -> torch.Tensor:
        o = self.offsets[k]
        return self.ids[o : o + self.counts[k]]


def _check_bounds(boundaries) -> tuple:
    bounds = tuple(int(b) for b in boundaries)
    if not bounds or bounds[0] < 1 or any(a >= b for a, b in zip(bounds, bounds[1:])):
        raise ValueError(f"boundaries must be non-empty, ascending, >= 1: {bounds}")
    if bounds[-1] > _I32_MAX:
        raise ValueError(f"boundaries must fit int32: {bounds}")
    return bounds


def _partition(lengths: torch.Tensor, bounds: tuple, ids: torch.Tensor | None, stream=None):
    """Launch K2; returns (ids_out, counts list, first bad index or -1)."""
    lib = _lib.load()
    n = lengths.numel()
    dev = lengths.device
    ws_bytes = lib.b2_strata_workspace_bytes(n)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    ids_out = torch.empty(n, dtype=torch.int32, device=dev)
    counts = torch.empty(len(bounds), dtype=torch.int64, device=dev)
    bad = torch.empty(1, dtype=torch.int64, device=dev)
    rc = lib.b2_strata_partition(
        lengths.data_ptr(), ids.data_ptr() if ids is not None else None, n,
        _lib.i32_array(bounds), len(bounds), ids_out.data_ptr(), counts.data_ptr(),
        bad.data_ptr(), ws.data_ptr(), ws_bytes, _lib.stream_ptr(stream),
    )
    _lib.check(rc)
    host = torch.cat([bad, counts]).cpu().tolist()  # one D2H: nb + 1 integers
    return ids_out, host[1:], host[0]


def _as_i32_device(x, what: str) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(x)))
    if t.dtype != torch.int32:
        if t.numel() and (int(t.max()) > _I32_MAX or int(t.min()) < -_I32_MAX - 1):
            raise ValueError(f"{what} must fit int32")
        t = t.to(torch.int32)
    return t.reshape(-1).to("cuda", non_blocking=True).contiguous()


def stratify_lengths(lengths, boundaries=DEFAULT_STRATUM_BOUNDARIES, ids=None, stream=None) -> DeviceStrata:
    """Tensor fast path of ``stratify``: lengths (and optional ids) -> DeviceStrata.

    ids default to 0..n-1.  Raises like the reference for an empty corpus, a
    sample beyond the last boundary (naming its id) or a length < 1.
    """
    bounds = _check_bounds(boundaries)
    _lib.load()
    lens = _as_i32_device(lengths, "lengths")
    n = lens.numel()
    if n == 0:
        raise ValueError("cannot stratify an empty corpus")
    idt = _as_i32_device(ids, "ids") if ids is not None else None
    ids_out, counts, bad = _partition(lens, bounds, idt, stream)
    if bad >= 0:
        length = int(lens[bad])
        sid = int(idt[bad]) if idt is not None else bad
        if length < 1:
            raise ValueError(f"sample length must be >= 1, got {length}")
        raise ValueError(
            f"sample id {sid} has length {length}, beyond the last stratum boundary {bounds[-1]}"
        )
    probs = tuple(int(c) / n for c in counts)
    return DeviceStrata(boundaries=bounds, ids=ids_out, counts=tuple(int(c) for c in counts), probs=probs)


def stratify_shards(lengths, shard_offsets: Sequence[int], boundaries=DEFAULT_STRATUM_BOUNDARIES,
                    stream=None) -> list:
    """Stratify every rank shard ``lengths[off[g]:off[g+1]]`` in one device pass.

    Equivalent to ``stratify_lengths`` on each shard (ids are shard-local
    indices); returns one ``DeviceStrata`` per shard (views into one buffer).
    """
    bounds = _check_bounds(boundaries)
    lib = _lib.load()
    lens = _as_i32_device(lengths, "lengths")
    offs = [int(o) for o in shard_offsets]
    if len(offs) < 2 or offs[0] != 0 or offs[-1] != lens.numel() or any(a >= b for a, b in zip(offs, offs[1:])):
        raise ValueError("shard_offsets must start at 0, end at len(lengths) and be strictly increasing")
    ns = len(offs) - 1
    dev = lens.device
    ws_bytes = lib.b2_strata_workspace_bytes(lens.numel())
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    ids_out = torch.empty(lens.numel(), dtype=torch.int32, device=dev)
    counts = torch.empty((ns, len(bounds)), dtype=torch.int64, device=dev)
    bad = torch.empty(ns, dtype=torch.int64, device=dev)
    rc = lib.b2_strata_partition_shards(
        lens.data_ptr(), None, _lib.i64_array(offs), ns, _lib.i32_array(bounds), len(bounds), ids_out.data_ptr(),
        counts.data_ptr(), bad.data_ptr(), ws.data_ptr(), ws_bytes, _lib.stream_ptr(stream))
    _lib.check(rc)
    host = torch.cat([bad, counts.reshape(-1)]).cpu().tolist()
    out = []
    for g in range(ns):
        if host[g] >= 0:
            i = host[g]
            length = int(lens[offs[g] + i])
            if length < 1:
                raise ValueError(f"sample length must be >= 1, got {length}")
            raise ValueError(f"sample id {i} has length {length}, beyond the last stratum boundary {bounds[-1]}")
        cnt = tuple(int(c) for c in host[ns + g * len(bounds): ns + (g + 1) * len(bounds)])
        n = offs[g + 1] - offs[g]
        out.append(DeviceStrata(boundaries=bounds, ids=ids_out[offs[g]:offs[g + 1]], counts=cnt,
                                probs=tuple(c / n for c in cnt)))
    return out


def stratify(samples: Sequence[Sample], boundaries=DEFAULT_STRATUM_BOUNDARIES) -> Strata:
    """Partition samples into strata by length, preserving input order (strata.py:61-83)."""
    bounds = _check_bounds(boundaries)
    if not samples:
        raise ValueError("cannot stratify an empty corpus")
    samples = list(samples)
    lens = np.fromiter((s.length for s in samples), dtype=np.int64, count=len(samples))
    # lengths beyond int32 are beyond every boundary: clamp, K2 reports them as bad
    lens32 = np.minimum(lens, _I32_MAX).astype(np.int32)
    _lib.load()
    dev_lens = torch.from_numpy(lens32).to("cuda", non_blocking=True)
    # the kernel partitions input slots; slots map back to the caller's Sample objects
    slots, counts, bad = _partition(dev_lens, bounds, None)
    if bad >= 0:
        s = samples[bad]
        raise ValueError(
            f"sample id {s.id} has length {s.length}, beyond the last stratum boundary {bounds[-1]}"
        )
    order = slots.cpu().numpy()
    buckets, o = [], 0
    for c in counts:
        buckets.append([samples[i] for i in order[o : o + c]])
        o += c
    total = len(samples)
    return Strata(boundaries=bounds, buckets=buckets, probs=tuple(len(p) / total for p in buckets))


def allocate_counts(probs: Sequence[float], local_batch: int) -> StratumAllocation:
    """Largest-remainder apportionment, ties to the lower stratum (strata.py:86-110)."""
    p = np.asarray(probs, dtype=float)
    if p.ndim != 1 or p.size == 0:
        raise ValueError("probs must be a non-empty 1-D sequence")
    if (p < 0).any():
        raise ValueError(f"negative probability in {probs}")
    if local_batch < 0:
        raise ValueError(f"local_batch must be >= 0, got {local_batch}")
    total = p.sum()
    if total <= 0:
        raise ValueError("probabilities sum to zero")
    quota = local_batch * p / total
    base = np.floor(quota).astype(int)
    extra = local_batch - int(base.sum())
    if extra:
        base[np.argsort(-(quota - base), kind="stable")[:extra]] += 1
    return StratumAllocation(tuple(int(c) for c in base), local_batch)


def draw_batch(strata: Strata, alloc: StratumAllocation, seed: int) -> list:
    """Draw alloc.counts[k] samples per stratum without replacement (strata.py:113-141).

    Host-side by design (numpy PCG64 stream = the reference's draws); pools
    shrink across calls and a dry stratum borrows from the nonempty stratum
    with the closest boundary.
    """
    if len(alloc.counts) != strata.num_strata:
        raise ValueError(
            f"allocation has {len(alloc.counts)} strata, corpus has {strata.num_strata}"
        )
    rng = np.random.default_rng(seed)
    out: list = []

    def pull(pool: list, take: int) -> None:
        if take == 0:
            return
        # swap-pop in descending index order keeps lower indices valid (:147-152)
        for i in sorted((int(i) for i in rng.choice(len(pool), size=take, replace=False)), reverse=True):
            out.append(pool[i])
            pool[i] = pool[-1]
            pool.pop()

    for k, need in enumerate(alloc.counts):
        take = min(need, len(strata.buckets[k]))
        pull(strata.buckets[k], take)
        short = need - take
        while short > 0:
            cands = [
                (abs(strata.boundaries[j] - strata.boundaries[k]), j)
                for j in range(strata.num_strata)
                if j != k and strata.buckets[j]
            ]
            if not cands:
                raise ValueError(
                    f"stratum {k + 1} exhausted and no other stratum can cover "
                    f"the remaining {short} sample(s)"
                )
            j = min(cands)[1]
            take = min(short, len(strata.buckets[j]))
            pull(strata.buckets[j], take)
            short -= take
    return out


class NativeDraws:
    """Bit-exact native port of draw_batch (strata.py:113-161) over mutable id pools (host C++).

    Same numpy PCG64 stream as the reference (SeedSequence -> PCG64 ->
    Generator.choice(replace=False)), same swap-pop and closest-boundary
    borrowing; differential-tested against numpy (tests/test_draws.py).  Runs
    on the host CPU like the reference's data loader, ~100x faster than the
    Python loop; `epoch` draws many steps in one call with the per-(key, step)
    seeds of seeding.derive_seed.
    """

    def __init__(self, pools, boundaries):
        import ctypes

        self.lib = _lib.load(require_device=False)
        bounds = [int(b) for b in boundaries]
        arrs = [np.asarray(p, dtype=np.int64).reshape(-1) for p in pools]
        if len(arrs) != len(bounds):
            raise ValueError(f"{len(arrs)} pools for {len(bounds)} boundaries")
        flat = np.ascontiguousarray(np.concatenate(arrs) if arrs else np.zeros(0, np.int64))
        sizes = np.array([a.size for a in arrs], dtype=np.int64)
        self.nstrata = len(bounds)
        h = ctypes.c_void_p()
        _lib.check(self.lib.b2_draws_create(ctypes.byref(h), flat.ctypes.data, sizes.ctypes.data, self.nstrata,
                                            np.asarray(bounds, dtype=np.int64).ctypes.data))
        self.handle = h

    def remaining(self) -> tuple:
        return tuple(int(self.lib.b2_draws_remaining(self.handle, k)) for k in range(self.nstrata))

    def _raise(self, err_k, err_s):
        raise ValueError(
            f"stratum {err_k.value} exhausted and no other stratum can cover the remaining {err_s.value} sample(s)"
        )

    def draw(self, counts, seed: int) -> np.ndarray:
        import ctypes

        c = np.asarray(counts, dtype=np.int64)
        if c.size != self.nstrata:
            raise ValueError(f"allocation has {c.size} strata, corpus has {self.nstrata}")
        out = np.empty(int(c.sum()), dtype=np.int64)
        ek, es = ctypes.c_int(0), ctypes.c_int64(0)
        rc = self.lib.b2_draw_batch(self.handle, c.ctypes.data, int(seed) & (2**64 - 1), out.ctypes.data,
                                    ctypes.byref(ek), ctypes.byref(es))
        if rc != 0:
            self._raise(ek, es)
        return out

    def epoch(self, counts, base_seed: int, key=(), first_step: int = 0, nsteps: int = 1):
        """Draw steps t = first_step.. with seed derive_seed(base_seed, *key, t); returns (ids[done, lb], done).

        Stops early (done < nsteps) at global exhaustion; the reference would
        raise there, callers decide.
        """
        import ctypes

        c = np.asarray(counts, dtype=np.int64)
        lb = int(c.sum())
        out = np.empty((int(nsteps), lb), dtype=np.int64)
        k = np.asarray(list(key), dtype=np.uint64)
        done = ctypes.c_int64(0)
        ek, es = ctypes.c_int(0), ctypes.c_int64(0)
        self.lib.b2_draw_epoch(self.handle, c.ctypes.data, int(base_seed), k.ctypes.data if k.size else None,
                               int(k.size), int(first_step), int(nsteps), out.ctypes.data, ctypes.byref(done),
                               ctypes.byref(ek), ctypes.byref(es))
        return out[: done.value], int(done.value)

    def close(self) -> None:
        if self.handle:
            self.lib.b2_draws_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def derive_seed(seed: int, *key: int) -> int:
    """seeding.py:18-21 (native)."""
    lib = _lib.load(require_device=False)
    k = np.asarray(key, dtype=np.uint64)
    return int(lib.b2_derive_seed(int(seed), k.ctypes.data if k.size else None, int(k.size)))
