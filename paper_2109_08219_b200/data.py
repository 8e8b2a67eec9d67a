"""Synthetic inputs for the B200 path (reference datasets: data.py:58-113).

``generate(dist, n, seed, device)`` fills a device buffer with the library's
counter-based generator (``dtopk_generate``, csrc/generate.cuh): value i
depends only on (seed, i), so any shard of a vector can be produced on its own
GPU without communication.  The integer distributions have a bit-exact numpy
twin (``generate_host``) used by the CPU tests; float distributions are
produced on the device and copied when a host copy is needed.

The reference's own host generators are kept with their names and draws
(``gen_uniform`` / ``gen_normal`` / ``gen_customized``, data.py:54-113: numpy
Philox, so a vector is a function of (seed, position) for a given numpy), and
``generate`` also accepts the reference's names "ud" / "nd" / "cd" (host
numpy result, reference semantics).  The DTKV vector file (data.py:116-161:
16-byte header "DTKV", version 1, u64 count, u32 little-endian payload) is
read window by window, which is how the partitioned run streams partitions
that are not resident (distributed.run_distributed, SURVEY.md section 8f rows
f1-f2).
"""

from __future__ import annotations

import numpy as np
import torch

import os
import struct

from . import _native
from .core import DtopkError

DISTS = {
    "uniform": (0, 0),
    "ascending": (1, 0),
    "all_equal": (2, 0x5A5A5A5A),
    "few_distinct": (3, 16),
    "normal_f32": (4, 0),
    "pareto_f32": (5, 1500),
    "nd_u32": (6, 0),
    "descending": (7, 0),
}
FLOAT_DISTS = {"normal_f32", "pareto_f32"}

_MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def generate(dist: str, n: int, seed: int = 0, device=None, *, param: int | None = None,
             offset: int = 0, k: int | None = None):
    """Device vector of ``n`` keys; ``offset`` shifts the counter (shards).

    The reference's dataset names "ud" / "nd" / "cd" (data.py:164-175) return
    the reference's host vectors instead (``k`` is required for "cd")."""
    if dist in GENERATORS:
        if dist == "cd":
            if k is None:
                raise ValueError("the cd distribution requires k")
            return gen_customized(n, k, seed)
        return GENERATORS[dist](n, seed)
    if dist not in DISTS:
        raise ValueError(f"unknown distribution {dist!r}; expected one of {sorted(DISTS)}")
    code, default = DISTS[dist]
    p = default if param is None else param
    if dist == "descending" and param is None:
        p = n - 1 + offset
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    dtype = torch.float32 if dist in FLOAT_DISTS else torch.uint32
    out = torch.empty(n, dtype=dtype, device=dev)
    lib = _native.load()
    if offset:
        # counter offset: generate the global vector's [offset, offset + n) window
        if code in (1,):
            p = p + offset
        elif code == 7:
            p = p - offset
        else:
            return _generate_window(code, n, seed, p, offset, dev, dtype)
    with torch.cuda.device(dev):
        st = lib.dtopk_generate(out.data_ptr(), n, code, seed, p, torch.cuda.current_stream(dev).cuda_stream)
    _native.check(st, "dtopk_generate")
    return out


def _generate_window(code, n, seed, p, offset, dev, dtype):
    # the kernel hashes (seed, i); a window is the tail of a longer run
    full = torch.empty(offset + n, dtype=dtype, device=dev)
    lib = _native.load()
    with torch.cuda.device(dev):
        st = lib.dtopk_generate(full.data_ptr(), offset + n, code, seed, p, torch.cuda.current_stream(dev).cuda_stream)
    _native.check(st, "dtopk_generate")
    return full[offset:].clone()


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def generate_host(dist: str, n: int, seed: int = 0, *, param: int | None = None, offset: int = 0) -> np.ndarray:
    """Bit-exact numpy twin of ``generate`` for the integer distributions."""
    code, default = DISTS[dist]
    p = default if param is None else param
    i = np.arange(offset, offset + n, dtype=np.uint64)
    if code == 1:
        return (i + np.uint64(p)).astype(np.uint32)
    if code == 7:
        q = (n - 1 + offset) if param is None else p
        return (np.uint64(q) - i).astype(np.uint32)
    if code == 2:
        return np.full(n, p, dtype=np.uint32)
    key = _splitmix64(np.array([np.uint64(seed) ^ np.uint64(0xD1B54A32D192ED03)]))[0]
    with np.errstate(over="ignore"):
        h = _splitmix64(i + key)
    hi = (h >> np.uint64(32)).astype(np.uint32)
    if code == 0:
        return hi
    if code == 3:
        return (hi % np.uint32(max(p, 1))).astype(np.uint32)
    raise ValueError(f"{dist} has no bit-exact host twin; generate on the device and copy")


# ---------------------------------------------------------------------------
# reference datasets (data.py:54-113) and the DTKV vector file (data.py:116-161)
# ---------------------------------------------------------------------------
MAGIC = b"DTKV"
VERSION = 1
_HEADER = struct.Struct("<4sIQ")
HEADER_SIZE = _HEADER.size  # 16 bytes
ELEMENT_SIZE = 4
NORMAL_MEAN = 10**8
NORMAL_STDDEV = 10.0
CD_LEVELS = 4      # 8-bit refinement levels of the adversarial construction
CD_BUCKETS = 256


class BadMagic(DtopkError):
    """The file does not start with the vector-file magic."""


class BadVersion(DtopkError):
    """The file's format version is unsupported."""


class TruncatedFile(DtopkError):
    """The file is shorter than its header says it should be."""


class InfeasibleN(DtopkError):
    """n (or k) is too small for the adversarial construction."""


def _philox(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def gen_uniform(n: int, seed: int) -> np.ndarray:
    """U[0, 2^32) draws (data.py:58-62)."""
    if n < 1:
        raise ValueError("n must be at least 1")
    return _philox(seed).integers(0, 2**32, size=n, dtype=np.uint32)


def gen_normal(n: int, seed: int) -> np.ndarray:
    """rint(N(1e8, 10)) clamped to u32 (data.py:65-75): heavy duplication, stresses ties."""
    if n < 1:
        raise ValueError("n must be at least 1")
    x = _philox(seed).normal(NORMAL_MEAN, NORMAL_STDDEV, size=n)
    return np.clip(np.rint(x), 0, 2**32 - 1).astype(np.uint32)


def gen_customized(n: int, k: int, seed: int) -> np.ndarray:
    """Adversarial vector for range refinement (data.py:78-113): one sentinel in
    every non-top 8-bit bucket of the first three levels, the rest uniform in
    the top chain [0xFFFFFF00, 2^32), positions shuffled.  Same draw order as
    the reference, so the same numpy gives the same bytes."""
    per_level = CD_BUCKETS - 1
    levels = CD_LEVELS - 1
    if n < 4 * CD_LEVELS * per_level:
        raise InfeasibleN(f"n={n} below {4 * CD_LEVELS * per_level}, too small for "
                          f"{CD_LEVELS} refinement levels of {CD_BUCKETS} buckets")
    cluster = n - levels * per_level
    if k > cluster:
        raise InfeasibleN(f"k={k} exceeds the dense cluster size {cluster}")
    rng = _philox(seed)
    parts, prefix = [], 0
    for lv in range(levels):
        sh = 32 - 8 * (lv + 1)
        lows = rng.integers(0, 1 << sh, size=per_level, dtype=np.uint64)
        parts.append((prefix | (np.arange(per_level, dtype=np.uint64) << sh) | lows).astype(np.uint32))
        prefix |= 0xFF << sh
    parts.append(rng.integers(prefix, 2**32, size=cluster, dtype=np.uint64).astype(np.uint32))
    return np.concatenate(parts)[rng.permutation(n)]


GENERATORS = {"ud": gen_uniform, "nd": gen_normal, "cd": gen_customized}


def write_vector(path, values) -> None:
    """Vector file with a little-endian u32 payload (data.py:116-121)."""
    if isinstance(values, torch.Tensor):
        values = values.detach().cpu().numpy()
    values = np.ascontiguousarray(values).ravel()
    if values.dtype != np.uint32:
        values = values.astype(np.uint32)
    with open(path, "wb") as f:
        f.write(_HEADER.pack(MAGIC, VERSION, values.size))
        values.astype("<u4", copy=False).tofile(f)


def read_header(path) -> int:
    """Validate a vector file's header; return its element count (data.py:124-140)."""
    size = os.path.getsize(path)
    if size < HEADER_SIZE:
        raise TruncatedFile(f"{path}: {size} bytes is shorter than the 16-byte header")
    with open(path, "rb") as f:
        magic, version, count = _HEADER.unpack(f.read(HEADER_SIZE))
    if magic != MAGIC:
        raise BadMagic(f"{path}: bad magic {magic!r}, expected {MAGIC!r}")
    if version != VERSION:
        raise BadVersion(f"{path}: unsupported version {version}, expected {VERSION}")
    if size != HEADER_SIZE + ELEMENT_SIZE * count:
        raise TruncatedFile(f"{path}: header promises {count} elements "
                            f"({HEADER_SIZE + ELEMENT_SIZE * count} bytes) but file has {size} bytes")
    return count


def read_vector(path, *, offset: int = 0, count: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """Read the [offset, offset + count) window of a vector file (data.py:143-161).

    ``out``: optional destination (e.g. a pinned host buffer viewed as numpy)
    so a streamed partition lands where the H2D copy reads it.
    """
    total = read_header(path)
    if count is None:
        count = total - offset
    if offset < 0 or count < 0 or offset + count > total:
        raise ValueError(f"window [{offset}, {offset + count}) outside vector of {total} elements")
    with open(path, "rb") as f:
        f.seek(HEADER_SIZE + ELEMENT_SIZE * offset)
        if out is None:
            data = np.fromfile(f, dtype="<u4", count=count)
        else:
            data = out[:count]
            got = f.readinto(memoryview(data.view(np.uint8)))
            if got != count * ELEMENT_SIZE:
                raise TruncatedFile(f"{path}: payload ended early inside the requested window")
            return data
    if data.size != count:
        raise TruncatedFile(f"{path}: payload ended early inside the requested window")
    return data.astype(np.uint32, copy=False)
