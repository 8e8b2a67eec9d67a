"""Synthetic inputs for the B200 path (reference datasets: data.py:58-113).

``generate(dist, n, seed, device)`` fills a device buffer with the library's
counter-based generator (``dtopk_generate``, csrc/generate.cuh): value i
depends only on (seed, i), so any shard of a vector can be produced on its own
GPU without communication.  The integer distributions have a bit-exact numpy
twin (``generate_host``) used by the CPU tests; float distributions are
produced on the device and copied when a host copy is needed.

The reference's own Philox generators (gen_uniform / gen_normal /
gen_customized) are numpy-version specific; golden fixtures made with them
live in tests/golden/.  The DTKV file format (data.py:116-161) is outside the
hot path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native

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
             offset: int = 0) -> torch.Tensor:
    """Device vector of ``n`` keys; ``offset`` shifts the counter (shards)."""
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
