"""CPU oracle for the Dr. Top-k hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this module.  It is the
checker, never the thing measured or shipped: the product path
(``paper_2109_08219_b200``) has no CPU fallback.

Two layers, both restating the reference package (paths under
``/root/reference/pkg/src/dtopk/``):

* ``libdtopk_oracle.so`` (``oracle/dtopk_oracle.c``), the fast C restatement
  of ``pipeline.dr_topk`` used at sizes up to 2^30;
* small pure-numpy restatements below, used to cross-check the C oracle.

Parity of both against the reference itself is pinned by the golden vectors in
``tests/golden/golden.npz`` (produced by ``tests/golden/make_golden.py`` from
the reference package in the build container).
"""

from __future__ import annotations

import ctypes
import math
import os
import pathlib
import subprocess

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
_SO = _HERE / "_build" / "libdtopk_oracle.so"
_lib = None


class OracleStats(ctypes.Structure):
    _fields_ = [
        ("delegate_vector_len", ctypes.c_uint64),
        ("concatenated_len", ctypes.c_uint64),
        ("fully_qualified_subranges", ctypes.c_uint64),
        ("partially_qualified_subranges", ctypes.c_uint64),
        ("elements_read", ctypes.c_uint64),
        ("elements_written", ctypes.c_uint64),
        ("theta", ctypes.c_uint32),
        ("threshold", ctypes.c_uint32),
        ("pool_len", ctypes.c_uint64),
    ]


def build() -> pathlib.Path:
    """Compile the C oracle with gcc (no reference sources are involved)."""
    _SO.parent.mkdir(parents=True, exist_ok=True)
    src = _HERE / "dtopk_oracle.c"
    if not _SO.exists() or _SO.stat().st_mtime < src.stat().st_mtime:
        subprocess.check_call(
            ["gcc", "-O3", "-march=native", "-fPIC", "-shared", "-pthread", "-o", str(_SO), str(src), "-lm"]
        )
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not _SO.exists():
            build()
        L = ctypes.CDLL(str(_SO))
        u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
        i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
        L.oracle_auto_alpha.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int]
        L.oracle_auto_alpha.restype = ctypes.c_int
        L.oracle_extract_delegates.argtypes = [u32p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, u32p]
        L.oracle_radix_threshold.argtypes = [u32p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
        L.oracle_radix_threshold.restype = ctypes.c_uint32
        L.oracle_dr_topk.argtypes = [u32p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, u32p, ctypes.POINTER(OracleStats)]
        L.oracle_dr_topk.restype = ctypes.c_int
        L.oracle_topk_indices.argtypes = [u32p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, u32p, i64p]
        L.oracle_f32_to_keys.argtypes = [u32p, ctypes.c_uint64, ctypes.c_int, u32p]
        L.oracle_dr_topk_partitioned.argtypes = [u32p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                                 ctypes.c_double, ctypes.c_int, u32p]
        L.oracle_dr_topk_partitioned.restype = ctypes.c_int
        L.oracle_generate_uniform.argtypes = [u32p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int]
        _lib = L
    return _lib


# ---------------------------------------------------------------------------
# key maps (float32 / smallest): the order-preserving bijection named in the
# reference README as the extension point (pkg/README.md:108-110)
# ---------------------------------------------------------------------------
def to_keys(v: np.ndarray, largest: bool = True) -> np.ndarray:
    v = np.ascontiguousarray(v)
    if v.dtype == np.float32:
        b = v.view(np.uint32)
        u = np.where(b >> np.uint32(31), ~b, b | np.uint32(0x80000000)).astype(np.uint32)
    else:
        u = v.astype(np.uint32, copy=False)
    return u if largest else ~u


def from_keys(u: np.ndarray, dtype, largest: bool = True) -> np.ndarray:
    u = np.asarray(u, dtype=np.uint32)
    if not largest:
        u = ~u
    if np.dtype(dtype) == np.float32:
        b = np.where(u & np.uint32(0x80000000), u ^ np.uint32(0x80000000), ~u).astype(np.uint32)
        return b.view(np.float32)
    return u


# ---------------------------------------------------------------------------
# C oracle wrappers
# ---------------------------------------------------------------------------
def auto_alpha(n: int, k: int, const_c: float = 3.0, beta: int = 2) -> int:
    return int(lib().oracle_auto_alpha(n, k, const_c, beta))


def extract_delegates(keys: np.ndarray, alpha: int, beta: int) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    s = -(-keys.size // (1 << alpha))
    out = np.empty(beta * s, dtype=np.uint32)
    lib().oracle_extract_delegates(keys, keys.size, alpha, beta, out)
    return out


def radix_threshold(vals: np.ndarray, k: int, skip_last: bool) -> int:
    vals = np.ascontiguousarray(vals, dtype=np.uint32)
    return int(lib().oracle_radix_threshold(vals, vals.size, k, int(skip_last), None))


def dr_topk(keys: np.ndarray, k: int, alpha: int, beta: int, skip_last: bool = True, direct: bool = False):
    """Values (non-increasing) and stats of pipeline.dr_topk on uint32 keys."""
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    out = np.empty(k, dtype=np.uint32)
    st = OracleStats()
    rc = lib().oracle_dr_topk(keys, keys.size, k, alpha, beta, int(skip_last), int(direct), out, ctypes.byref(st))
    if rc != 0:
        raise ValueError(f"oracle_dr_topk failed rc={rc}")
    return out, st


def topk_with_indices(keys: np.ndarray, k: int, kth: int | None = None):
    """(keys, indices) of the top-k under (key desc, index asc) -- the
    reference tie rule of kernels._extract_exact (kernels.py:83-96) on V."""
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    if kth is None:
        kth = radix_threshold(keys, k, False)
    ok = np.empty(k, dtype=np.uint32)
    oi = np.empty(k, dtype=np.int64)
    lib().oracle_topk_indices(keys, keys.size, k, kth, ok, oi)
    return ok, oi


def generate_uniform(n: int, seed: int = 0, offset: int = 0, threads: int | None = None) -> np.ndarray:
    """Host twin of data.generate('uniform', ...) (bit-exact), multi-threaded."""
    out = np.empty(n, dtype=np.uint32)
    lib().oracle_generate_uniform(out, n, seed, offset, threads or cpu_count())
    return out


def dr_topk_partitioned(keys: np.ndarray, k: int, workers: int, beta: int = 2, const_c: float = 3.0) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint32)
    out = np.empty(k, dtype=np.uint32)
    rc = lib().oracle_dr_topk_partitioned(keys, keys.size, k, beta, const_c, workers, out)
    if rc != 0:
        raise ValueError(f"oracle_dr_topk_partitioned failed rc={rc}")
    return out


# ---------------------------------------------------------------------------
# pure-numpy restatements (small sizes) used to cross-check the C oracle
# ---------------------------------------------------------------------------
def np_extract_delegates(keys: np.ndarray, alpha: int, beta: int) -> np.ndarray:
    """delegate.py:132-155: zero padded rows, top-beta per row, non-increasing."""
    w = 1 << alpha
    rows = -(-keys.size // w)
    grid = np.zeros(rows * w, dtype=np.uint32)
    grid[: keys.size] = keys
    grid = grid.reshape(rows, w)
    padded = np.concatenate([grid, np.zeros((rows, beta), dtype=np.uint32)], axis=1)
    return np.sort(padded, axis=1)[:, ::-1][:, :beta].reshape(-1).copy()


def np_radix_threshold(vals: np.ndarray, k: int, skip_last: bool) -> int:
    """kernels.py:130-165, 8-bit digits."""
    vals = np.asarray(vals, dtype=np.uint32)
    bits, mask, rem = 0, 0, k
    for p in range(4 - int(skip_last)):
        shift = 24 - 8 * p
        live = vals if mask == 0 else vals[(vals & np.uint32(mask)) == np.uint32(bits)]
        hist = np.bincount((live >> np.uint32(shift)) & np.uint32(255), minlength=256)
        at_least = np.cumsum(hist[::-1])[::-1]
        d = int(np.flatnonzero(at_least >= rem)[-1])
        rem -= int(at_least[d + 1]) if d < 255 else 0
        bits |= d << shift
        mask |= 255 << shift
    if not skip_last:
        return bits
    return int(vals[vals >= np.uint32(bits)].min())


def np_topk_with_indices(keys: np.ndarray, k: int):
    """O(n log n) restatement: lexsort by (key desc, index asc)."""
    keys = np.asarray(keys, dtype=np.uint32)
    order = np.lexsort((np.arange(keys.size), ~keys))[:k]
    return keys[order], order.astype(np.int64)


def cpu_count() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def log2(x: float) -> float:
    return math.log2(x)
