"""Standalone top-k / k-selection operators (mirror of dtopk.kernels).

``radix_topk`` keeps the reference signature (kernels.py:109-165) and returns
``(selected_values, selected_tags, threshold)``; on the GPU it is the direct
path of ``dtopk_select`` (exact radix select over the whole input with
11/11/10-bit digits, ordered emit, stable sort), so the selected elements are
the reference's ``_extract_exact`` choice (kernels.py:83-96): every element
above the k-th, then ties in scan order.  ``bucket_topk`` / ``bitonic_topk``
are not rebuilt (out of scope, identical value
multisets), and the reference oracles ``sort_and_choose`` / ``heap_topk`` live
in ``oracle/`` as test infrastructure only.
"""

from __future__ import annotations

from typing import NamedTuple

import torch

from . import _device, _native
from .core import InvalidK, PipelineConfig, WorkloadStats

RADIX_BITS = 8  # reference digit width (kernels.py:39); the device uses 11/11/10
RADIX_PASSES = 32 // RADIX_BITS


class KeyedEntry(NamedTuple):
    """A selection key with an opaque payload (kernels.py:44-51)."""

    value: int
    tag: int


def kth_largest(keys: torch.Tensor, k: int) -> int:
    """Exact k-th largest of a uint32 CUDA tensor (``dtopk_kth_largest``)."""
    lib = _native.load()
    keys = _device._aligned(_device._torch_u32(keys))
    n = keys.numel()
    if not 1 <= k <= n:
        raise InvalidK(f"k={k} outside [1, {n}]")
    wsb = int(lib.dtopk_workspace_bytes(n, k, 0, 1, 1))
    ws = torch.empty(wsb, dtype=torch.uint8, device=keys.device)
    out = torch.empty(1, dtype=torch.uint32, device=keys.device)
    with torch.cuda.device(keys.device):
        st = lib.dtopk_kth_largest(keys.data_ptr(), n, k, out.data_ptr(), ws.data_ptr(), wsb,
                                   torch.cuda.current_stream(keys.device).cuda_stream)
    _native.check(st, "dtopk_kth_largest")
    return int(out.view(torch.int32).item()) & 0xFFFFFFFF


def radix_topk(values, k, *, skip_last=False, digit_bits=RADIX_BITS, tags=None, stats=None, states=None,
               largest: bool = True):
    """Exact (or skip_last-relaxed) radix top-k (kernels.py:109-165).

    Returns (selected_values, selected_tags, threshold) in the reference's order
    and dtype: elements above the k-th in scan order, then the k-th's ties in
    scan order (``_extract_exact``), or every element >= the relaxed edge in
    scan order (``_extract_at_least``); values in the input dtype.  ``digit_bits`` is validated like the reference but
    the device always uses its own 11/11/10 digits; ``states`` is not
    recorded on the device.
    """
    if digit_bits < 1 or 32 % digit_bits:
        raise ValueError(f"digit_bits={digit_bits} must divide 32")
    del states
    _native.load()
    dv = _device.to_device(values)
    if not 1 <= k <= dv.n:
        raise InvalidK(f"k={k} outside [1, {dv.n}]")
    from .pipeline import DrTopK

    # alpha = 0 resolves to direct_fallback (core.py:173): the whole input is the pool
    cfg = PipelineConfig(k=k, alpha=0, auto_alpha=False, largest=largest)
    plan = DrTopK(dv.n, cfg, dv.code, dv.out_dtype, dv.device, timed=False)
    assert plan.cfg.direct_fallback
    with torch.cuda.device(dv.device):
        plan.launch(dv.keys)
        hdr = plan.header()
    # _extract_exact's order (kernels.py:83-96): every element above the k-th in
    # scan order, then the k-th's ties in scan order.  The device answer is
    # ordered (key desc, index asc), so its ties already close it in index
    # order; only the strictly-better head is re-sorted by index.
    kth = int(hdr.kth_key)
    bits = dv.keys.view(torch.int32)
    keyv = plan.values.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    if dv.code == _native.DTYPE_F32:
        keyv = torch.where(keyv >> 31 == 1, keyv ^ 0xFFFFFFFF, keyv | 0x80000000)
    if not largest:
        keyv = 0xFFFFFFFF - keyv
    n_gt = int((keyv > kth).sum().item())
    idx = torch.cat([torch.sort(plan.indices[:n_gt]).values, plan.indices[n_gt:]])
    sel = bits[idx].view(plan.values.dtype) if plan.values.dtype != torch.int32 else bits[idx]
    threshold = _device.key_to_value(kth, dv.code, largest)
    if skip_last:
        # kernels.py:161-164: every element at or above the lower edge of the
        # 256-wide bucket holding the k-th key; threshold = their minimum.
        keys64 = dv.keys.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        if dv.code == _native.DTYPE_F32 or not largest:
            raise NotImplementedError("skip_last relaxation is defined on uint32-largest keys only")
        edge = int(hdr.kth_key) & 0xFFFFFF00
        mask = keys64 >= edge
        idx = torch.nonzero(mask).flatten()  # _extract_at_least: scan order
        sel = bits[idx].view(torch.uint32) if plan.values.dtype == torch.uint32 else bits[idx]
        threshold = int((keys64[idx]).min().item())
    if stats is not None:
        stats.add_read(2 * dv.n)
        stats.add_written(int(sel.numel()))
    sel_tags = None
    if tags is not None:
        t = tags if isinstance(tags, torch.Tensor) else torch.as_tensor(tags)
        t = t.to(idx.device)
        t = t.to(torch.int64) if t.dtype == torch.uint32 else t
        sel_tags = _device.to_caller(t[idx], dv.kind)
    return _device.to_caller(sel, dv.kind), sel_tags, threshold
