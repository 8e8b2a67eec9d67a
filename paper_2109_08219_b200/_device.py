"""Input/output plumbing between caller containers and device buffers.

The reference accepts anything ``np.asarray(v, dtype=uint32)`` accepts
(core.py:45-52) and returns numpy arrays.  The drop-in keeps that contract for
host inputs (numpy, lists, CPU tensors: copied to HBM once, results copied
back) and adds a zero-copy path for CUDA tensors (results stay on device).

Key dtypes: uint32 (and int32, reinterpreted bit for bit as numpy's
``astype(uint32)`` does) run on the uint32 key path; float32 runs on the
float32 key path (order-preserving bit map inside the kernels).  Any other
integer dtype is wrapped to uint32 like the reference coercion.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .core import ELEMENT_DTYPE, EmptyInput


@dataclass
class DeviceVector:
    keys: torch.Tensor  # 1-D contiguous, 16-byte aligned, on CUDA
    code: int  # _native.DTYPE_U32 / DTYPE_F32
    out_dtype: torch.dtype  # dtype of returned values
    kind: str  # "numpy" | "torch_cpu" | "torch_cuda"
    h2d_bytes: int = 0

    @property
    def n(self) -> int:
        return int(self.keys.numel())

    @property
    def device(self) -> torch.device:
        return self.keys.device


def _aligned(t: torch.Tensor) -> torch.Tensor:
    t = t.reshape(-1)
    if not t.is_contiguous():
        t = t.contiguous()
    if t.data_ptr() % 16:
        t = t.clone()
    return t


def _torch_u32(t: torch.Tensor) -> torch.Tensor:
    if t.dtype == torch.uint32:
        return t
    if t.dtype == torch.int32:
        return t.view(torch.uint32)
    if t.dtype in (torch.int64, torch.int16, torch.int8, torch.uint8, torch.bool, torch.uint16):
        return (t.to(torch.int64) & 0xFFFFFFFF).to(torch.uint32)
    raise TypeError(f"unsupported key dtype {t.dtype}; use uint32, int32 or float32")


def to_device(v, device: torch.device | None = None) -> DeviceVector:
    """Coerce a caller's vector into an aligned device key buffer."""
    if isinstance(v, torch.Tensor):
        if v.numel() == 0:
            raise EmptyInput("input vector must hold at least one element")
        if v.is_cuda:
            if v.dtype == torch.float32:
                return DeviceVector(_aligned(v), _native.DTYPE_F32, torch.float32, "torch_cuda")
            return DeviceVector(_aligned(_torch_u32(v)), _native.DTYPE_U32, v.dtype if v.dtype == torch.int32 else torch.uint32, "torch_cuda")
        dev = device or torch.device("cuda", torch.cuda.current_device())
        if v.dtype == torch.float32:
            host = v.reshape(-1).contiguous()
            code, odt = _native.DTYPE_F32, torch.float32
        else:
            host = _torch_u32(v.reshape(-1)).contiguous()
            code, odt = _native.DTYPE_U32, (torch.int32 if v.dtype == torch.int32 else torch.uint32)
        d = host.to(dev, non_blocking=False)
        return DeviceVector(_aligned(d), code, odt, "torch_cpu", h2d_bytes=host.numel() * 4)
    arr = np.asarray(v)
    if arr.dtype == np.float32:
        host = np.ascontiguousarray(arr.ravel())
        code, odt = _native.DTYPE_F32, torch.float32
    else:
        host = np.ascontiguousarray(np.asarray(v, dtype=ELEMENT_DTYPE).ravel())
        code, odt = _native.DTYPE_U32, torch.uint32
    if host.size == 0:
        raise EmptyInput("input vector must hold at least one element")
    dev = device or torch.device("cuda", torch.cuda.current_device())
    d = torch.from_numpy(host).to(dev)
    return DeviceVector(_aligned(d), code, odt, "numpy", h2d_bytes=host.size * 4)


@dataclass
class HostVector:
    host: torch.Tensor  # 1-D contiguous CPU tensor (uint32 or float32 bits as stored)
    code: int
    out_dtype: torch.dtype
    kind: str  # "numpy" | "torch_cpu"

    @property
    def n(self) -> int:
        return int(self.host.numel())


def host_view(v) -> HostVector | None:
    """A host input as a flat CPU tensor without copying (None for CUDA tensors)."""
    if isinstance(v, torch.Tensor):
        if v.is_cuda:
            return None
        if v.numel() == 0:
            raise EmptyInput("input vector must hold at least one element")
        if v.dtype == torch.float32:
            return HostVector(v.reshape(-1).contiguous(), _native.DTYPE_F32, torch.float32, "torch_cpu")
        odt = torch.int32 if v.dtype == torch.int32 else torch.uint32
        return HostVector(_torch_u32(v.reshape(-1)).contiguous(), _native.DTYPE_U32, odt, "torch_cpu")
    arr = np.asarray(v)
    if arr.dtype == np.float32:
        host, code, odt = np.ascontiguousarray(arr.ravel()), _native.DTYPE_F32, torch.float32
    else:
        host = np.ascontiguousarray(np.asarray(v, dtype=ELEMENT_DTYPE).ravel())
        code, odt = _native.DTYPE_U32, torch.uint32
    if host.size == 0:
        raise EmptyInput("input vector must hold at least one element")
    return HostVector(torch.from_numpy(host), code, odt, "numpy")


# Streamed host input (reference residency / reload plan,
# distributed.py:97-137): ranges of STREAM_RANGE keys go host -> pinned staging
# (parallel CPU copy, pageable inputs only) -> HBM on a copy stream, and K1
# reduces each range as soon as it has landed, so the H2D stream is the only
# serial cost.  Two staging buffers per device, allocated once.
STREAM_MIN = 1 << 24
STREAM_RANGE = 1 << 24  # keys per range (64 MiB), a multiple of the 2048-key K1 chunk
_staging: dict = {}


def staging_buffers(device: torch.device):
    st = _staging.get(device)
    if st is None:
        bufs = [torch.empty(STREAM_RANGE, dtype=torch.int32, pin_memory=True) for _ in range(2)]
        evs = [None, None]
        st = _staging[device] = (bufs, evs, torch.cuda.Stream(device))
    return st


def to_caller(t: torch.Tensor, kind: str):
    """Return a result in the caller's container kind."""
    if kind == "torch_cuda":
        return t
    if kind == "torch_cpu":
        return t.cpu()
    return t.cpu().numpy()


def key_to_value(key: int, code: int, largest: bool):
    """Host-side inverse key map for the scalar threshold (no device read)."""
    u = key & 0xFFFFFFFF
    if not largest:
        u = ~u & 0xFFFFFFFF
    if code == _native.DTYPE_F32:
        b = (u ^ 0x80000000) if (u & 0x80000000) else (~u & 0xFFFFFFFF)
        return float(np.array([b], dtype=np.uint32).view(np.float32)[0])
    return int(u)
