"""Monte-Carlo balance engine on B200 (drop-in for ``ddpsim.mcsim``).

Reference: ``mcsim.py`` — every trial draws one global batch, forms the
per-GPU assignment and records the min / max per-GPU token count; averages
over trials give the balance table (``run_balance_experiment`` :79-81,
``run_ablation`` :84-110, ``_run`` :284-300).

Split by where each piece is cheapest, bit-exact with the reference:

* **draws** (device, one warp per trial: ``b2_mc_draw_device``; or host C++
  threads: ``b2_mc_draw``) port numpy's ``SeedSequence(seed, spawn_key=(t,))``
  -> PCG64 -> ``Generator.choice(replace=False)`` for every trial
  (``derive_rng``, seeding.py:8-16; ``_stratified_matrix`` :166-180;
  ``_draw_uniform`` :146-151).  Trials are independent.  The device path
  covers numpy's Floyd branch (every paper configuration); the tail-shuffle
  branch (a large share of a pool) stays on the host threads.
* **token counts** (device): ``b2_mc_token_counts`` sorts each node's pool
  (LOCAL_PRESORT), or the whole batch (GLOBAL_PRESORT), deals raster / snake,
  sums per GPU in int64 and reduces min / max per trial, all trials in one
  launch (:182-213).
* **aggregation** (host): the reference's own numpy expressions on the
  int64 min / max arrays (:290-306), so the float statistics match bit for bit.

With host draws, draw and count overlap chunk by chunk (host threads fill
pinned buffer i+1 while the GPU counts chunk i).  ``PACKING`` needs ``pack_corpus``, which is
outside this build's scope, and raises ``NotImplementedError``.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, replace
from enum import Enum

import numpy as np
import torch

from . import _lib
from .balance import ScanPattern
from .seqdata import MAX_SEQ_LEN, Topology
from .strata import DEFAULT_STRATUM_BOUNDARIES, allocate_counts, derive_seed, stratify_lengths

_STRATEGY_CODE = {"none": 0, "stratified": 1, "local_presort": 2, "global_presort": 3}


class Strategy(str, Enum):
    """mcsim.py:31-40."""

    NONE = "none"
    GLOBAL_PRESORT = "global_presort"
    PACKING = "packing"
    LOCAL_PRESORT = "local_presort"
    STRATIFIED = "stratified"


@dataclass(frozen=True)
class BalanceExperiment:
    """mcsim.py:43-67.  ``samples`` may also be an int array of lengths (ids 0..N-1)."""

    strategy: Strategy
    topo: Topology
    samples: object
    seed: int
    local_batch: int = 16
    trials: int = 100_000
    scan: ScanPattern = ScanPattern.RASTER
    pack_limit: int = 2
    max_seq_len: int = MAX_SEQ_LEN
    stratum_boundaries: tuple = DEFAULT_STRATUM_BOUNDARIES

    def __post_init__(self):
        object.__setattr__(self, "strategy", Strategy(self.strategy))
        object.__setattr__(self, "scan", ScanPattern(self.scan))
        if not isinstance(self.samples, (np.ndarray, torch.Tensor)):
            object.__setattr__(self, "samples", tuple(self.samples))
        if self.trials < 1:
            raise ValueError(f"trials must be >= 1, got {self.trials}")
        if self.local_batch < 1:
            raise ValueError(f"local_batch must be >= 1, got {self.local_batch}")
        if self.pack_limit < 1:
            raise ValueError(f"pack_limit must be >= 1, got {self.pack_limit}")
        if len(self.samples) == 0:
            raise ValueError("experiment needs a non-empty corpus")


@dataclass(frozen=True)
class BalanceStats:
    """Averages over trials of the per-trial min/max per-GPU token count (mcsim.py:70-80)."""

    trials: int
    avg_min: float
    avg_max: float
    avg_range: float
    stderr_min: float
    stderr_max: float
    stderr_range: float


def _lengths_of(samples) -> np.ndarray:
    if isinstance(samples, torch.Tensor):
        return samples.detach().cpu().numpy().astype(np.int64).reshape(-1)
    if isinstance(samples, np.ndarray):
        return samples.astype(np.int64).reshape(-1)
    return np.fromiter((s.length for s in samples), dtype=np.int64, count=len(samples))


@dataclass
class _Prepared:
    pools_dev: torch.Tensor  # int32 lengths of the draw pools, concatenated (device)
    pool_sizes: np.ndarray   # int64 per pool
    counts: np.ndarray       # int64 per-GPU draws per pool
    max_len: int
    _pools_host: np.ndarray | None = None

    @property
    def pools(self) -> np.ndarray:
        """Host copy of the pools (for the host draw threads), made on first use."""
        if self._pools_host is None:
            self._pools_host = np.ascontiguousarray(self.pools_dev.cpu().numpy())
        return self._pools_host


def _prepare(exp: BalanceExperiment) -> _Prepared:
    """mcsim._prepare (:122-143), plus the exhaustion checks of the draws."""
    if exp.strategy is Strategy.PACKING:
        raise NotImplementedError("the PACKING strategy needs pack_corpus, outside this build's scope (SURVEY §2)")
    lengths = _lengths_of(exp.samples)
    G, b = exp.topo.total_gpus, exp.local_batch
    if lengths.min() < 1:
        raise ValueError(f"sample length must be >= 1, got {int(lengths.min())}")
    uniform = exp.strategy in (Strategy.NONE, Strategy.GLOBAL_PRESORT)
    if uniform and b * G > lengths.size:  # _draw_uniform :147-150
        raise ValueError(f"corpus exhausted within a trial: needs {b * G} samples, corpus has {lengths.size}")
    lens_dev = torch.from_numpy(lengths.astype(np.int32)).cuda()
    if exp.strategy in (Strategy.STRATIFIED, Strategy.LOCAL_PRESORT):
        ds = stratify_lengths(lens_dev, exp.stratum_boundaries)  # K2, stable per stratum (strata.py:61-83)
        pools = lens_dev[ds.ids.long()]  # the strata's lengths, stratum after stratum (device gather)
        sizes = np.asarray(ds.counts, dtype=np.int64)
        counts = np.asarray(allocate_counts(ds.probs, b).counts, dtype=np.int64)
        for c, n in zip(counts, sizes):  # _stratified_matrix :170-177
            need = int(c) * G
            if need and need > n:
                raise ValueError(
                    f"corpus exhausted within a trial: a stratum holds {int(n)} "
                    f"samples but the trial needs {need}"
                )
    else:
        pools = lens_dev
        sizes = np.asarray([lengths.size], dtype=np.int64)
        counts = np.asarray([b], dtype=np.int64)
    return _Prepared(pools_dev=pools.contiguous(), pool_sizes=sizes, counts=counts, max_len=int(lengths.max()))


def draw_trials(exp: BalanceExperiment, first_trial: int, ntrials: int, out: np.ndarray | torch.Tensor | None = None,
                prep: _Prepared | None = None, threads: int | None = None):
    """Host draws of trials [first, first+n): int32 [n, b*G] (the (b, G) matrices, row-major)."""
    prep = prep if prep is not None else _prepare(exp)
    lib = _lib.load(require_device=False)
    G, b = exp.topo.total_gpus, exp.local_batch
    if out is None:
        out = np.empty((ntrials, b * G), dtype=np.int32)
    ptr = out.data_ptr() if isinstance(out, torch.Tensor) else out.ctypes.data
    nthreads = threads or max(1, len(os.sched_getaffinity(0)))
    _lib.check(lib.b2_mc_draw(prep.pools.ctypes.data, prep.pool_sizes.ctypes.data, int(prep.pool_sizes.size),
                              prep.counts.ctypes.data, G, int(exp.seed) & (2**64 - 1), int(first_trial),
                              int(ntrials), int(nthreads), ptr))
    return out


def draw_trials_device(exp: BalanceExperiment, first_trial: int, ntrials: int, out: torch.Tensor | None = None,
                       prep: _Prepared | None = None, pools: torch.Tensor | None = None, stream=None):
    """Device draws of trials [first, first+n) into a CUDA int32 [n, b*G] tensor
    (``b2_mc_draw_device``: the same bits as ``draw_trials``).  Returns None when
    a stratum falls in numpy's tail-shuffle branch (host draws only)."""
    prep = prep if prep is not None else _prepare(exp)
    lib = _lib.load()
    G, b = exp.topo.total_gpus, exp.local_batch
    if pools is None:
        pools = prep.pools_dev
    if out is None:
        out = torch.empty((ntrials, b * G), dtype=torch.int32, device="cuda")
    rc = lib.b2_mc_draw_device(pools.data_ptr(), prep.pool_sizes.ctypes.data, int(prep.pool_sizes.size),
                               prep.counts.ctypes.data, G, int(exp.seed) & (2**64 - 1), int(first_trial),
                               int(ntrials), out.data_ptr(), _lib.stream_ptr(stream))
    if rc == _lib.B2_ERR_UNSUPPORTED:
        return None
    _lib.check(rc)
    return out


def trial_token_counts(exp: BalanceExperiment, mat: torch.Tensor, max_len: int, counts: bool = False,
                       stream=None):
    """Device: [n, b*G] int32 length matrices -> (mins, maxs[, counts [n, G]]) int64 on the device."""
    lib = _lib.load()
    n = mat.shape[0]
    G, b = exp.topo.total_gpus, exp.local_batch
    dev = mat.device
    mins = torch.empty(n, dtype=torch.int64, device=dev)
    maxs = torch.empty(n, dtype=torch.int64, device=dev)
    cnt = torch.empty((n, G), dtype=torch.int64, device=dev) if counts else None
    bad = torch.empty(1, dtype=torch.int32, device=dev)
    scan = _lib.B2_SCAN_SNAKE if exp.scan is ScanPattern.SNAKE else _lib.B2_SCAN_RASTER
    _lib.check(lib.b2_mc_token_counts(mat.data_ptr(), n, b, G, exp.topo.gpus_per_node,
                                      _STRATEGY_CODE[exp.strategy.value], scan, int(max_len),
                                      cnt.data_ptr() if cnt is not None else None, mins.data_ptr(),
                                      maxs.data_ptr(), bad.data_ptr(), _lib.stream_ptr(stream)))
    return (mins, maxs, cnt, bad)


def _stats(trials: int, mins: np.ndarray, maxs: np.ndarray) -> BalanceStats:
    """mcsim._run aggregation (:290-300) and _stderr (:303-306), same numpy calls."""
    ranges = maxs - mins
    return BalanceStats(
        trials=trials,
        avg_min=float(mins.mean()),
        avg_max=float(maxs.mean()),
        avg_range=float(ranges.mean()),
        stderr_min=_stderr(mins),
        stderr_max=_stderr(maxs),
        stderr_range=_stderr(ranges),
    )


def _stderr(values: np.ndarray) -> float:
    if values.size < 2:
        return 0.0
    return float(values.std(ddof=1) / math.sqrt(values.size))


def run_trials(exp: BalanceExperiment, chunk: int = 4096, threads: int | None = None, draws: str = "auto"):
    """All trials: (mins, maxs) int64 host arrays.

    draws="device" (and "auto" when every stratum is in numpy's Floyd branch):
    draws and counts both on the GPU, chunk by chunk.  draws="host" (and the
    "auto" fallback): host-thread draws of chunk i+1 overlap the device
    counts of chunk i (two pinned buffers, one copy stream)."""
    prep = _prepare(exp)
    if draws in ("auto", "device"):
        res = _run_trials_device(exp, prep, chunk)
        if res is not None:
            return res
        if draws == "device":
            raise _lib.B2Error("device draws unsupported for this experiment (numpy tail-shuffle branch)")
    G, b = exp.topo.total_gpus, exp.local_batch
    T = exp.trials
    chunk = max(1, min(chunk, T))
    host = [torch.empty((chunk, b * G), dtype=torch.int32, pin_memory=True) for _ in range(2)]
    dev = [torch.empty((chunk, b * G), dtype=torch.int32, device="cuda") for _ in range(2)]
    done = [torch.cuda.Event(), torch.cuda.Event()]
    mins = torch.empty(T, dtype=torch.int64, device="cuda")
    maxs = torch.empty(T, dtype=torch.int64, device="cuda")
    bads = []
    stream = torch.cuda.current_stream()
    for i, t0 in enumerate(range(0, T, chunk)):
        n = min(chunk, T - t0)
        k = i & 1
        done[k].synchronize()  # buffer k's previous copy has finished
        draw_trials(exp, t0, n, out=host[k][:n], prep=prep, threads=threads)
        dev[k][:n].copy_(host[k][:n], non_blocking=True)
        mn, mx, _, bad = trial_token_counts(exp, dev[k][:n], prep.max_len, stream=stream)
        mins[t0:t0 + n].copy_(mn, non_blocking=True)
        maxs[t0:t0 + n].copy_(mx, non_blocking=True)
        bads.append(bad)
        done[k].record(stream)
    if int(torch.stack(bads).max()) != 0:
        raise ValueError("a drawn length is outside [1, max length] (corrupt corpus)")
    return mins.cpu().numpy(), maxs.cpu().numpy()


def _run_trials_device(exp: BalanceExperiment, prep: _Prepared, chunk: int):
    G, b = exp.topo.total_gpus, exp.local_batch
    T = exp.trials
    chunk = max(1, min(chunk, T))
    pools = prep.pools_dev
    mat = torch.empty((chunk, b * G), dtype=torch.int32, device="cuda")
    mins = torch.empty(T, dtype=torch.int64, device="cuda")
    maxs = torch.empty(T, dtype=torch.int64, device="cuda")
    bads = []
    for t0 in range(0, T, chunk):
        n = min(chunk, T - t0)
        if draw_trials_device(exp, t0, n, out=mat[:n], prep=prep, pools=pools) is None:
            return None
        mn, mx, _, bad = trial_token_counts(exp, mat[:n], prep.max_len)
        mins[t0:t0 + n].copy_(mn)
        maxs[t0:t0 + n].copy_(mx)
        bads.append(bad)
    if int(torch.stack(bads).max()) != 0:
        raise ValueError("a drawn length is outside [1, max length] (corrupt corpus)")
    return mins.cpu().numpy(), maxs.cpu().numpy()


def run_balance_experiment(exp: BalanceExperiment, chunk: int = 4096, threads: int | None = None) -> BalanceStats:
    """Run all trials of one experiment and aggregate the balance stats (mcsim.py:79-81)."""
    mins, maxs = run_trials(exp, chunk=chunk, threads=threads)
    return _stats(exp.trials, mins, maxs)


def run_ablation(base: BalanceExperiment, chunk: int = 4096, threads: int | None = None) -> list:
    """Step-by-step balance table (mcsim.py:84-110), rows on derive_seed(base.seed, i)."""
    if base.strategy is not Strategy.LOCAL_PRESORT:
        raise ValueError(
            f"ablation is defined for the local_presort lineage, got {base.strategy.value}"
        )
    rows = (
        ("none", Strategy.NONE, ScanPattern.RASTER),
        ("+stratification", Strategy.STRATIFIED, ScanPattern.RASTER),
        ("+local_presorting", Strategy.LOCAL_PRESORT, ScanPattern.RASTER),
        ("+snake_scanning", Strategy.LOCAL_PRESORT, ScanPattern.SNAKE),
        ("global_presort", Strategy.GLOBAL_PRESORT, ScanPattern.RASTER),
    )
    out = []
    for i, (label, strategy, scan) in enumerate(rows):
        exp = replace(base, strategy=strategy, scan=scan, seed=derive_seed(base.seed, i))
        out.append((label, run_balance_experiment(exp, chunk=chunk, threads=threads)))
    return out
