"""ctypes binding of the C-ABI library ``_native/libb2ddp.so`` (include/b2ddp.h).

There is deliberately no CPU fallback: if the library is missing or no CUDA
device is visible, every hot-path call raises.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import os

# B2_LIB_PATH: load another build of the same library (A/B measurements under tools/)
LIB_PATH = Path(os.environ.get("B2_LIB_PATH") or Path(__file__).resolve().parent / "_native" / "libb2ddp.so")

B2_OK, B2_ERR_INVALID, B2_ERR_CUDA, B2_ERR_INDIVISIBLE, B2_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
B2_F32, B2_BF16, B2_F64 = 0, 1, 2
B2_SCAN_RASTER, B2_SCAN_SNAKE = 0, 1

# every symbol include/b2ddp.h declares, with its ctypes signature
_P, _I, _I64, _D, _SZ = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_size_t
SIGNATURES = {
    "b2_version": (C.c_char_p, []),
    "b2_last_error": (C.c_char_p, []),
    "b2_clip_workspace_bytes": (_SZ, []),
    "b2_clip_workspace_init": (_I, [_P, _SZ, _P]),
    "b2_bucket_clip_cast": (
        _I,
        [_P, _I, _P, _I, _P, _P, _P, _I, _D, _D, _P, _P, _P, _P, _SZ, _I, _P],
    ),
    "b2_weighted_mean": (_I, [_P, _I, _I64, _I64, _I64, _P, _P, _I, _P, _I, _P]),
    "b2_nccl_unique_id": (_I, [_P, C.c_char_p]),
    "b2_comm_create": (_I, [C.POINTER(C.c_void_p), _I, _I, _P, C.c_char_p]),
    "b2_comm_destroy": (_I, [_P]),
    "b2_allreduce_avg": (_I, [_P, _P, _I64, _I, _P]),
    "b2_bucket_clip_allreduce": (
        _I,
        [_P, _P, _I, _P, _I, _P, _P, _I, _D, _P, _P, _P, _SZ, _P, _P],
    ),
    "b2_p2p_flag_bytes": (_SZ, []),
    "b2_ipc_export": (_I, [_P, _P, C.POINTER(C.c_int64)]),
    "b2_ipc_import": (_I, [_P, _I64, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "b2_ipc_close": (_I, [_P]),
    "b2_bucket_clip_allreduce_p2p": (
        _I,
        [_P, _P, _P, _I, _I, _P, _P, _I, _D, _P, _P, _P, _SZ, _P],
    ),
    "b2_bucket_clip_allreduce_p2p_dtype": (
        _I,
        [_P, _P, _I, _P, _I, _I, _P, _P, _I, _D, _P, _P, _P, _SZ, _P],
    ),
    "b2_derive_seed": (C.c_uint64, [C.c_uint64, _P, _I]),
    "b2_draws_create": (_I, [C.POINTER(C.c_void_p), _P, _P, _I, _P]),
    "b2_draws_destroy": (_I, [_P]),
    "b2_draws_remaining": (_I64, [_P, _I]),
    "b2_draw_batch": (_I, [_P, _P, C.c_uint64, _P, C.POINTER(C.c_int), C.POINTER(C.c_int64)]),
    "b2_draw_epoch": (
        _I,
        [_P, _P, C.c_uint64, _P, _I, _I64, _I64, _P, C.POINTER(C.c_int64), C.POINTER(C.c_int),
         C.POINTER(C.c_int64)],
    ),
    "b2_bucket_clip_allreduce_nvls": (
        _I,
        [_P, _P, _P, _P, _I, _I, _P, _P, _I, _D, _P, _P, _P, _SZ, _P],
    ),
    "b2_strata_workspace_bytes": (_SZ, [_I64]),
    "b2_strata_partition": (_I, [_P, _P, _I64, _P, _I, _P, _P, _P, _P, _SZ, _P]),
    "b2_strata_partition_shards": (_I, [_P, _P, _P, _I, _P, _I, _P, _P, _P, _P, _SZ, _P]),
    "b2_presort_deal": (
        _I,
        [_P, _P, _I64, _I, _I, _I, C.c_int32, C.c_int32, _P, _P, _P, _P, _P],
    ),
    "b2_presort_workspace_bytes": (_SZ, [_I64, _I, C.c_int32, C.c_int32, _I]),
    "b2_presort_sort_deal": (
        _I,
        [_P, _P, _I64, _I, _I, _I, C.c_int32, C.c_int32, _P, _P, _P, _P, _P, _SZ, _P],
    ),
    "b2_set_spin_timeout": (_I, [_D]),
    "b2_get_spin_timeout": (_D, []),
    "b2_mc_draw": (_I, [_P, _P, _I, _P, _I, C.c_uint64, _I64, _I64, _I, _P]),
    "b2_mc_token_counts": (_I, [_P, _I64, _I, _I, _I, _I, _I, C.c_int32, _P, _P, _P, _P, _P]),
    "b2_mc_draw_device": (_I, [_P, _P, _I, _P, _I, C.c_uint64, _I64, _I64, _P, _P]),
}

_lock = threading.Lock()
_lib = None


class B2Error(RuntimeError):
    """A C-ABI call failed (CUDA error or unsupported size)."""


def load(require_device: bool = True):
    """Load the library once; raise loudly when it (or a GPU) is missing."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise B2Error(
                        f"CUDA library {LIB_PATH} is not built; run "
                        "`python -c 'import __graft_entry__ as g; g.build()'`"
                    )
                lib = C.CDLL(str(LIB_PATH))
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = lib
    if require_device:
        import torch

        if not torch.cuda.is_available():
            raise B2Error("no CUDA device visible: the b2ddp hot paths have no CPU fallback")
    return _lib


def check(rc: int) -> None:
    if rc == B2_OK:
        return
    msg = _lib.b2_last_error().decode() if _lib is not None else "unknown error"
    if rc in (B2_ERR_INVALID, B2_ERR_INDIVISIBLE):
        raise ValueError(msg)
    raise B2Error(f"b2ddp error {rc}: {msg}")


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def i64_array(values):
    vals = [int(v) for v in values]
    return (C.c_int64 * max(1, len(vals)))(*vals)


def i32_array(values):
    vals = [int(v) for v in values]
    return (C.c_int32 * max(1, len(vals)))(*vals)
