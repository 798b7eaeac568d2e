"""B200-native hot paths of arXiv 2402.02447 behind the reference ``ddpsim`` API.

H1 (bucket-wise clip before allreduce): ``gradsync`` + ``ddp`` (fused
NVLink kernel, NCCL side stream, DDP comm hook) + ``reducer`` (Algorithm 1 on a
model's gradients, without DDP).  H2 (stratified local presort): ``strata`` +
``balance``; the Monte-Carlo balance engine in ``mcsim``.  All data passes run in ``_native/libb2ddp.so`` (sm_100a); see
DESIGN.md.  Names mirror ``ddpsim/__init__.py:14-103`` for the in-scope paths.
"""

from .balance import (
    Assignment,
    ScanPattern,
    assign_global_presort,
    assign_local_presort,
    presort_deal,
    presort_workspace_bytes,
    sort_shard,
)
from .gradsync import (
    BucketClipper,
    ClipConfig,
    ClipMode,
    GradientState,
    allreduce_mean,
    capped_bucket_layout,
    clip_by_norm,
    equal_bucket_layout,
    gradient_state_from_dict,
    sync_after,
    sync_before,
    sync_bucketwise,
    sync_bucketwise_host,
    synchronize,
)
from .seqdata import (
    DEFAULT_BIN_BOUNDARIES,
    DEFAULT_BIN_PROBS,
    MAX_SEQ_LEN,
    LengthDistribution,
    Sample,
    Topology,
    generate_corpus,
    generate_lengths,
)
from .strata import (
    DeviceStrata,
    Strata,
    StratumAllocation,
    allocate_counts,
    draw_batch,
    stratify,
    stratify_lengths,
    stratify_shards,
    NativeDraws,
    derive_seed,
)

from .mcsim import BalanceExperiment, BalanceStats, Strategy, run_ablation, run_balance_experiment
from .reducer import BucketwiseReducer

__version__ = "0.1.0"

__all__ = [
    "Assignment", "ScanPattern", "assign_global_presort", "assign_local_presort", "presort_deal",
    "presort_workspace_bytes", "sort_shard",
    "BucketClipper", "ClipConfig", "ClipMode", "GradientState", "allreduce_mean",
    "capped_bucket_layout", "clip_by_norm", "equal_bucket_layout", "gradient_state_from_dict",
    "sync_after", "sync_before", "sync_bucketwise", "sync_bucketwise_host", "synchronize",
    "DEFAULT_BIN_BOUNDARIES", "DEFAULT_BIN_PROBS", "MAX_SEQ_LEN", "LengthDistribution",
    "Sample", "Topology", "generate_corpus", "generate_lengths",
    "DeviceStrata", "Strata", "StratumAllocation", "allocate_counts", "draw_batch",
    "stratify", "stratify_lengths", "stratify_shards", "NativeDraws", "derive_seed",
    "BalanceExperiment", "BalanceStats", "Strategy", "run_ablation", "run_balance_experiment",
    "BucketwiseReducer",
]
