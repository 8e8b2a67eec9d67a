"""Delegate extraction (mirror of dtopk.delegate, delegate.py:1-191).

Both entry points run the sm_100a K1 kernel (``dtopk_extract_delegates``):
one TMA-streamed pass that emits, for every 2**alpha subrange, its beta
largest keys, non-increasing, with zero padding when the tail subrange holds
fewer than beta elements (delegate.py:132-139).  The reference's blocked
variant for alpha <= 5 (delegate.py:158-191) is the same kernel: on the GPU
small subranges are handled by the lane-per-subrange mapping of K1.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _device, _native
from .core import InvalidBeta, WorkloadStats

SMALL_SUBRANGE_ALPHA = 5  # delegate.py:29
BLOCK_SUBRANGES = 32  # delegate.py:30 (a warp)


@dataclass(frozen=True)
class DelegateVector:
    """Per-subrange top-beta keys and their subrange ids (delegate.py:33-55).

    ``values`` are keys (for uint32-largest inputs: the values themselves);
    ``tags`` = repeat(arange(S), beta).  Containers follow the input kind.
    """

    values: object
    tags: object
    beta: int
    subrange_count: int

    def __len__(self) -> int:
        return int(self.values.shape[0])


def _check_args(n: int, alpha: int, beta: int) -> int:
    width = 1 << alpha if alpha >= 0 else 0
    if alpha < 0 or width > n:
        raise ValueError(f"alpha={alpha} must satisfy 0 <= alpha and 2**alpha <= {n}")
    if not 1 <= beta < width:
        raise InvalidBeta(f"beta={beta} must satisfy 1 <= beta < 2**alpha={width}")
    return width


def extract_delegates(v, alpha: int, beta: int, *, stats: WorkloadStats | None = None,
                      largest: bool = True) -> DelegateVector:
    """Top-beta delegates of every 2**alpha subrange (delegate.py:142-155)."""
    _native.load()
    dv = _device.to_device(v)
    _check_args(dv.n, alpha, beta)
    lib = _native.load()
    s = -(-dv.n // (1 << alpha))
    out = torch.empty(beta * s, dtype=torch.uint32, device=dv.device)
    wsb = int(lib.dtopk_workspace_bytes(dv.n, 1, alpha, beta, 0))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dv.device)
    with torch.cuda.device(dv.device):
        st = lib.dtopk_extract_delegates(dv.keys.data_ptr(), dv.n, dv.code, int(largest), alpha, beta,
                                         out.data_ptr(), ws.data_ptr(), wsb,
                                         torch.cuda.current_stream(dv.device).cuda_stream)
    _native.check(st, "dtopk_extract_delegates")
    tags = torch.arange(s, dtype=torch.int64, device=dv.device).repeat_interleave(beta).to(torch.uint32)
    if stats is not None:
        stats.add_read(dv.n)
        stats.add_written(out.numel())
    return DelegateVector(_device.to_caller(out, dv.kind), _device.to_caller(tags, dv.kind), beta, s)


def extract_delegates_blocked(v, alpha: int, beta: int, *, stats: WorkloadStats | None = None,
                              blocks_per_batch: int = 512, largest: bool = True) -> DelegateVector:
    """Small-subrange entry point (delegate.py:158-191); same device kernel."""
    if alpha > SMALL_SUBRANGE_ALPHA:
        raise ValueError(f"blocked extraction is for alpha <= {SMALL_SUBRANGE_ALPHA}, got {alpha}")
    del blocks_per_batch  # batching is a CPU cache-blocking knob; K1 streams the whole vector
    return extract_delegates(v, alpha, beta, stats=stats, largest=largest)
