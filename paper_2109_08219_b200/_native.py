"""ctypes binding of libdtopk.so (the C ABI declared in include/dtopk.h).

The library is the product: there is no CPU fallback.  If the shared object
is missing, or no CUDA device is visible, every entry point raises
``NativeUnavailable`` loudly instead of computing anything on the host.
"""

from __future__ import annotations

import ctypes
import pathlib
import threading

import os

# DTOPK_LIB overrides the library path (used to A/B kernel variants in profiling runs)
LIB_PATH = pathlib.Path(os.environ.get("DTOPK_LIB") or pathlib.Path(__file__).resolve().parent / "_lib" / "libdtopk.so")

OK = 0
EMPTY_INPUT = 1
INVALID_K = 2
INVALID_BETA = 3
INVALID_ARG = 4
WORKSPACE_TOO_SMALL = 5
CUDA_ERROR = 6
UNSUPPORTED = 7

DTYPE_U32 = 0
DTYPE_F32 = 1
FLAG_EXACT_STATS = 1
FLAG_DELEGATES_DONE = 2

PATH_SELECT = 1
PATH_MERGE = 2
PATH_DIRECT = 3


class NativeUnavailable(RuntimeError):
    """libdtopk.so is missing or cannot run (no CUDA device)."""


class DtopkResult(ctypes.Structure):
    """Mirror of dtopk_result (include/dtopk.h)."""

    _fields_ = [
        ("k_out", ctypes.c_uint64),
        ("candidate_subranges", ctypes.c_uint64),
        ("fully_qualified", ctypes.c_uint64),
        ("partially_qualified", ctypes.c_uint64),
        ("concatenated_len", ctypes.c_uint64),
        ("concat_skipped_fq", ctypes.c_uint64),
        ("elements_reread", ctypes.c_uint64),
        ("pool_gt", ctypes.c_uint64),
        ("pool_eq", ctypes.c_uint64),
        ("delegate_bucket", ctypes.c_uint64),
        ("theta_local", ctypes.c_uint32),
        ("theta", ctypes.c_uint32),
        ("kth_key", ctypes.c_uint32),
        ("path", ctypes.c_uint32),
        ("theta_slot", ctypes.c_int64),
        ("filtered", ctypes.c_uint32),
        ("filter_fallback", ctypes.c_uint32),
    ]


EXPORTS = {
    "dtopk_workspace_bytes": (ctypes.c_size_t, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "dtopk_result_offset": (ctypes.c_size_t, []),
    "dtopk_select": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
         ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
         ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p],
    ),
    "dtopk_select_begin": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
         ctypes.c_uint32, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p],
    ),
    "dtopk_select_finish": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
         ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
         ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p],
    ),
    "dtopk_extract_delegates": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p],
    ),
    "dtopk_kth_largest": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
         ctypes.c_void_p],
    ),
    "dtopk_plan_create": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
         ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
         ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)],
    ),
    "dtopk_plan_launch": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "dtopk_plan_kernels": (None, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_ulonglong), ctypes.POINTER(ctypes.c_ulonglong)]),
    "dtopk_plan_destroy": (None, [ctypes.c_void_p]),
    "dtopk_event_create": (ctypes.c_void_p, []),
    "dtopk_event_destroy": (None, [ctypes.c_void_p]),
    "dtopk_event_elapsed_ms": (ctypes.c_float, [ctypes.c_void_p, ctypes.c_void_p]),
    "dtopk_generate": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_void_p]),
    "dtopk_delegates_range": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
         ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p],
    ),
    "dtopk_stage_workspace_bytes": (ctypes.c_size_t, [ctypes.c_uint64]),
    "dtopk_qualify": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
         ctypes.c_void_p],
    ),
    "dtopk_concat": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64,
         ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p],
    ),
    "dtopk_min_at_least": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p,
                                          ctypes.c_void_p]),
    "dtopk_merge_tmp_pairs": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_uint64]),
    "dtopk_merge_lists": (
        ctypes.c_int,
        [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
    ),
    "dtopk_dsel_init": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]),
    "dtopk_dsel_hist": (
        ctypes.c_int,
        [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int,
         ctypes.c_void_p, ctypes.c_void_p],
    ),
    "dtopk_dsel_digit": (
        ctypes.c_int,
        [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_void_p],
    ),
    "dtopk_dsel_place": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
    ),
    "dtopk_launch_count": (ctypes.c_ulonglong, []),
    "dtopk_num_sms": (ctypes.c_int, []),
    "dtopk_version": (ctypes.c_char_p, []),
}

_lock = threading.Lock()
_lib = None


def load(require_cuda: bool = True):
    """Load libdtopk.so (cached).  Raises NativeUnavailable when absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeUnavailable(
                    f"{LIB_PATH} is missing: build it with `make` or `python -c 'import __graft_entry__ as g; g.build()'`"
                )
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in EXPORTS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_cuda:
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailable("dtopk needs a CUDA device (sm_100a); there is no CPU fallback")
    return _lib


def check(status: int, what: str) -> None:
    if status == OK:
        return
    from .core import EmptyInput, InvalidBeta, InvalidK

    msg = f"{what}: dtopk status {status}"
    if status == EMPTY_INPUT:
        raise EmptyInput(msg)
    if status == INVALID_K:
        raise InvalidK(msg)
    if status == INVALID_BETA:
        raise InvalidBeta(msg)
    if status == INVALID_ARG:
        raise ValueError(msg)
    if status == UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)
