"""Sharded top-k across the GPUs of one node (reference: distributed.py).

The reference runs one ``dr_topk`` per partition on in-process threads and
gathers ``k`` values per worker to a coordinator that sorts them
(distributed.py:140-251; the paper's MPI gather).  Here one
process drives one GPU (``torch.distributed``, NCCL over NVLink/NVSwitch):

1. every rank owns a contiguous shard (``plan``/``shard_bounds``: equal
   partitions, distributed.py:97-131) and runs K1-K2 locally
   (``dtopk_select_begin``) -> theta_r = kth(D_r), an int64 in device memory;
2. ``all_reduce(MAX)`` of theta_r (8 bytes): every theta_r <= kth(shard r) <=
   kth(V), so max_r theta_r is a valid global filter (the exchange the paper
   disabled on MPI, is ~10 us on NVLink);
3. each rank finishes (``dtopk_select_finish``) with theta* and emits at most
   k (value, global index) pairs ordered (key desc, index asc);
4. ``all_gather`` of the counts and the fixed-size candidate buffers, then an
   exact device top-k over the rank-ordered concatenation.  Shards are
   contiguous in rank order, so position order among equal keys is global
   index order and the tie rule (lowest index first) is preserved.

The per-rank compute is injectable (``LocalOps``) so the exchange/merge logic
is exercised by world-size-2 ``gloo`` tests on CPU; the product uses
``DeviceOps`` (sm_100a library) with NCCL.
"""

from __future__ import annotations

import math
import queue
import threading
import time
from dataclasses import dataclass, field, replace

import numpy as np
import torch
import torch.distributed as dist

from .core import InvalidK, PipelineConfig, TopKResult, WorkloadStats, validate_config


class WorkerFailed(RuntimeError):
    """A rank failed; the run is aborted (distributed.py:47-48)."""


@dataclass(frozen=True)
class Partition:
    index: int
    offset: int
    length: int
    resident: bool


@dataclass(frozen=True)
class PartitionPlan:
    n: int
    partition_len: int
    partitions: tuple
    assignments: dict

    def worker_count(self) -> int:
        return len(self.assignments)


DEFAULT_MAX_RESIDENT = 1 << 26  # distributed.py:43 (desk-scale cap of the CPU reference)


def plan(n: int, k: int, workers: int, max_resident: int = DEFAULT_MAX_RESIDENT) -> PartitionPlan:
    """Partition arithmetic of the reference (distributed.py:97-131)."""
    if workers < 1:
        raise ValueError("workers must be at least 1")
    if n < 1:
        raise ValueError("n must be at least 1")
    plen = math.ceil(n / workers) if workers * max_resident >= n else max_resident
    if k > plen:
        raise InvalidK(f"k={k} exceeds the partition length {plen}")
    parts, assign = [], {w: [] for w in range(workers)}
    for i in range(math.ceil(n / plen)):
        w = i % workers
        parts.append(Partition(i, i * plen, min(plen, n - i * plen), not assign[w]))
        assign[w].append(i)
    return PartitionPlan(n, plen, tuple(parts), assign)


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """[offset, offset + length) of rank's contiguous equal shard."""
    plen = math.ceil(n / world)
    lo = min(n, rank * plen)
    return lo, min(n, lo + plen) - lo


# ---------------------------------------------------------------------------
class LocalOps:
    """Per-rank compute used by ``sharded_topk`` (device or test stand-in)."""

    def begin(self, shard, cfg: PipelineConfig):  # -> (state, theta tensor int64[1])
        raise NotImplementedError

    def finish(self, state, theta: torch.Tensor, index_offset: int):  # -> (values, indices) of <= k pairs
        raise NotImplementedError

    def merge(self, values, indices, k: int, largest: bool):  # exact top-k of the concatenation
        raise NotImplementedError


class DeviceOps(LocalOps):
    """The product path: libdtopk.so on this rank's GPU."""

    def begin(self, shard, cfg):
        from . import _device, _native
        from .pipeline import DrTopK

        dv = _device.to_device(shard)
        p = DrTopK(dv.n, cfg, dv.code, dv.out_dtype, dv.device, timed=False)
        c = p.cfg
        s = torch.cuda.current_stream(dv.device)
        if c.direct_fallback:
            return (p, dv, True), None
        st = p.lib.dtopk_select_begin(dv.keys.data_ptr(), dv.n, dv.code, c.k, int(c.largest), c.alpha, c.beta,
                                      p.flags, p.ws.data_ptr(), p.ws_bytes, s.cuda_stream, None)
        _native.check(st, "dtopk_select_begin")
        off = _native.DtopkResult.theta_slot.offset
        theta = p.ws[off:off + 8].view(torch.int64)
        return (p, dv, False), theta

    def finish(self, state, theta, index_offset):
        from . import _native

        p, dv, direct = state
        c = p.cfg
        s = torch.cuda.current_stream(dv.device)
        if direct:
            p.launch(dv.keys, index_offset=index_offset)
        else:
            st = p.lib.dtopk_select_finish(
                dv.keys.data_ptr(), dv.n, dv.code, c.k, int(c.largest), c.alpha, c.beta, p.flags,
                theta.data_ptr() if theta is not None else None, p.values.data_ptr(), p.indices.data_ptr(),
                int(index_offset), p.ws.data_ptr(), p.ws_bytes, s.cuda_stream, None)
            _native.check(st, "dtopk_select_finish")
        hdr = p.header()
        k_out = int(hdr.k_out)
        return p.values[:k_out], p.indices[:k_out]

    def merge(self, values, indices, k, largest):
        from .pipeline import dr_topk

        r = dr_topk(values, PipelineConfig(k=k, alpha=0, auto_alpha=False, largest=largest))
        return r.values, indices[r.indices]


def sharded_topk(shard, n_total: int, k: int, cfg: PipelineConfig | None = None, *, group=None,
                 index_offset: int | None = None, exchange_theta: bool = True,
                 ops: LocalOps | None = None) -> TopKResult:
    """Global top-k of a vector sharded contiguously over the ranks of ``group``.

    Every rank passes its own shard (``shard_bounds`` layout unless
    ``index_offset`` is given) and receives the global answer.
    """
    from .core import EmptyInput

    ops = ops or DeviceOps()
    cfg = cfg or PipelineConfig(k=k)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n_local = int(shard.numel())
    if index_offset is None:
        index_offset, _ = shard_bounds(n_total, world, rank)
    # global validation, identical on every rank, before any collective
    if n_total < 1:
        raise EmptyInput("input vector must hold at least one element")
    if not 1 <= k <= n_total:
        raise InvalidK(f"k={k} outside [1, {n_total}]")
    validate_config(replace(cfg, k=k), n_total)
    k_local = min(k, n_local)
    dev = _dev_of(shard)
    state = theta = err = None
    lcfg = cfg
    if n_local > 0:
        try:
            lcfg = validate_config(replace(cfg, k=k_local), n_local)
            state, theta = ops.begin(shard, lcfg)
        except Exception as exc:  # surfaced like the reference's WorkerFailed (distributed.py:238-241)
            err = exc
    # a rank that failed must not leave its peers blocked in a collective:
    # every rank learns of any failure before the exchange
    flag = torch.tensor([1 if err is not None else 0], dtype=torch.int64, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    if int(flag.item()):
        if err is not None:
            raise WorkerFailed(f"rank {rank} failed in begin: {err!r}") from err
        raise WorkerFailed("another rank failed in begin")
    # Every rank must join the collective; direct-path and empty ranks contribute theta = 0.
    t = theta if theta is not None else torch.zeros(1, dtype=torch.int64, device=dev)
    if exchange_theta:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    if n_local > 0:
        vals, idx = ops.finish(state, t if (theta is not None and exchange_theta) else theta, index_offset)
    else:
        vdt = torch.float32 if shard.dtype == torch.float32 else torch.uint32
        vals = torch.empty(0, dtype=vdt, device=dev)
        idx = torch.empty(0, dtype=torch.int64, device=dev)
    # all_gather counts, then fixed-size candidate buffers
    cnt = torch.tensor([vals.numel()], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    width = max(counts) if counts else 0
    vbuf = torch.zeros(width, dtype=vals.dtype, device=dev)
    ibuf = torch.zeros(width, dtype=torch.int64, device=dev)
    vbuf[: vals.numel()] = vals
    ibuf[: idx.numel()] = idx
    vg = [torch.empty_like(vbuf) for _ in range(world)]
    ig = [torch.empty_like(ibuf) for _ in range(world)]
    dist.all_gather(_as_gatherable(vg), _as_gatherable([vbuf])[0], group=group)
    dist.all_gather(ig, ibuf, group=group)
    cat_v = torch.cat([g[:c] for g, c in zip(vg, counts)])
    cat_i = torch.cat([g[:c] for g, c in zip(ig, counts)])
    values, indices = ops.merge(cat_v, cat_i, k, cfg.largest)
    stats = WorkloadStats()
    stats.device = {"gathered_pairs": int(sum(counts)), "gathered_bytes": int(sum(counts)) * (vals.element_size() + 8),
                    "theta_global": int(t.item()) if exchange_theta else None}
    thr = values[-1].item() if hasattr(values, "item") else values[-1]
    return TopKResult(values=values, threshold=thr, stats=stats, indices=indices)


class ShardedTopK:
    """Planned ``sharded_topk`` for one rank (fixed shard size, k, config, dtype).

    The benchmark and serving path: workspaces and buffers are allocated once,
    a step never synchronises the host, and with the NCCL backend the whole
    step can be captured in one CUDA graph (``capture``).  Per step, on the
    current stream:

    1. K1-K2 (``dtopk_select_begin``) -> theta_r in the workspace's int64 slot;
    2. ``all_reduce(MAX)`` of that slot in place (``exchange_theta``; ranks on
       the direct path or with an empty shard contribute 0 from a zeroed slot);
    3. K3.. (``dtopk_select_finish`` with theta*) writes <= k_r (value, global
       index) pairs ordered (key desc, index asc) straight into this rank's
       send buffer ``[count | indices | value bits]``;
    4. merge="gather": ONE ``all_gather`` of the send buffers, then
       ``dtopk_merge_lists`` -- a tree of pairwise merge-path rounds on the
       device -- takes the exact first k pairs of the rank lists.  Shards are
       contiguous in rank order, so on equal keys the lower rank (= lower
       global index) comes first: the tie rule holds without a sort.
       merge="select" (default for k_local > 2^16 on more than one rank,
       SURVEY.md section 8e step 5): a distributed radix select over the
       candidates (``dtopk_dsel_*``: 3 histogram all-reduces + one all_gather
       of per-rank (above, equal) counts) decides every rank's contribution;
       each rank writes its pairs into its slots of a zeroed k-slot buffer,
       one all_reduce(SUM) assembles the answer and ``dtopk_merge_lists``
       merges the rank segments.  ~16k bytes per rank instead of 12*world*k.

    Every rank validates the global shape (n_total, k, cfg) identically before
    any collective, and every rank joins every collective whatever its shard
    (ragged last shard, empty shard, direct-path shard): the gather width is
    the global k_local = min(k, ceil(n_total / world)).
    """

    def __init__(self, shard: torch.Tensor, n_total: int, k: int, cfg: PipelineConfig | None = None, *,
                 group=None, index_offset: int | None = None, exchange_theta: bool = True,
                 merge: str = "auto"):
        from . import _device, _native
        from .core import EmptyInput
        from .pipeline import DrTopK

        cfg = cfg or PipelineConfig(k=k)
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        # global validation: identical on every rank, before any collective
        if n_total < 1:
            raise EmptyInput("input vector must hold at least one element")
        if not 1 <= k <= n_total:
            raise InvalidK(f"k={k} outside [1, {n_total}]")
        validate_config(replace(cfg, k=k), n_total)  # InvalidBeta / backend errors on every rank alike
        if merge not in ("auto", "gather", "select"):
            raise ValueError(f"unknown merge {merge!r}")
        if not isinstance(shard, torch.Tensor) or not shard.is_cuda:
            raise ValueError("ShardedTopK needs the shard resident on this rank's GPU")
        self.lib = _native.load()
        dev = shard.device
        self.device = dev
        self.n_local = int(shard.numel())
        if index_offset is None:
            index_offset, _ = shard_bounds(n_total, self.world, self.rank)
        self.index_offset = int(index_offset)
        self.k = int(k)
        w = self.world
        self.kl = min(self.k, -(-int(n_total) // w))  # global gather width
        self.k_loc = min(self.kl, self.n_local)
        self.exchange_theta = exchange_theta
        if shard.dtype == torch.float32:
            code, out_dtype = _native.DTYPE_F32, torch.float32
        else:
            code, out_dtype = _native.DTYPE_U32, torch.uint32
        self.code, self.out_dtype = code, out_dtype
        self.largest = bool(cfg.largest)
        self.local = None
        self.dv = None
        if self.n_local > 0:
            self.dv = _device.to_device(shard)
            self.lcfg = validate_config(replace(cfg, k=self.k_loc), self.n_local)
            self.local = DrTopK(self.n_local, self.lcfg, code, out_dtype, dev, timed=False)
        else:
            self.lcfg = None
        kl = self.kl
        # send buffer (int64 words): [count, 0, indices[kl], value bits[kl] as u32 pairs]
        self.pw = 2 + kl + (kl + 1) // 2
        self.send = torch.zeros(self.pw, dtype=torch.int64, device=dev)
        self.s_idx = self.send[2:2 + kl]
        self.s_val = self.send[2 + kl:].view(torch.int32)[:kl]
        self.direct = self.local is not None and self.lcfg.direct_fallback
        if self.local is not None and not self.direct:
            ws = self.local.ws
            off = _native.DtopkResult.theta_slot.offset
            self.theta = ws[off:off + 8].view(torch.int64)
        else:
            self.theta = torch.zeros(1, dtype=torch.int64, device=dev)
        if self.local is not None:
            koff = _native.DtopkResult.k_out.offset
            self.kout = self.local.ws[koff:koff + 8].view(torch.int64)
        if merge == "auto":
            merge = "select" if w > 1 and kl > (1 << 16) else "gather"
        self.merge_mode = merge
        self.values = torch.empty(self.k, dtype=out_dtype, device=dev)
        self.indices = torch.empty(self.k, dtype=torch.int64, device=dev)
        nl = w
        tmp_pairs = int(self.lib.dtopk_merge_tmp_pairs(nl, self.k))
        self.tmp_val = torch.empty(max(1, tmp_pairs), dtype=torch.int32, device=dev)
        self.tmp_idx = torch.empty(max(1, tmp_pairs), dtype=torch.int64, device=dev)
        self.tmp_len = torch.empty(2 * nl, dtype=torch.int64, device=dev)
        if merge == "gather":
            self.gathered = torch.empty(w * self.pw, dtype=torch.int64, device=dev)
        else:
            self.state = torch.empty(2, dtype=torch.int64, device=dev)
            self.hist = torch.empty(_SEL_BINS, dtype=torch.int64, device=dev)
            self.gt_eq = torch.zeros(2, dtype=torch.int64, device=dev)
            self.g_cnt = torch.empty(2 * w, dtype=torch.int64, device=dev)
            self.seg = torch.empty(2 * w, dtype=torch.int64, device=dev)
            self.slots = torch.empty(2 * self.k, dtype=torch.int64, device=dev)
        self.graph = None

    # -- one step ----------------------------------------------------------
    def _local(self, keys, s) -> None:
        from . import _native

        p, c, lib = self.local, self.lcfg, self.lib
        kl = self.k_loc
        if self.direct:
            if self.exchange_theta:
                self.theta.zero_()
                dist.all_reduce(self.theta, op=dist.ReduceOp.MAX, group=self.group)
            p.launch(keys, s, index_offset=self.index_offset)
            self.s_val[:kl].copy_(p.values.view(torch.int32)[:kl])
            self.s_idx[:kl].copy_(p.indices[:kl])
            self.send[0:1].fill_(kl)
            return
        _native.check(lib.dtopk_select_begin(keys.data_ptr(), self.n_local, self.code, c.k, int(c.largest), c.alpha,
                                             c.beta, p.flags, p.ws.data_ptr(), p.ws_bytes, s.cuda_stream, None),
                      "dtopk_select_begin")
        if self.exchange_theta:
            dist.all_reduce(self.theta, op=dist.ReduceOp.MAX, group=self.group)
        _native.check(lib.dtopk_select_finish(
            keys.data_ptr(), self.n_local, self.code, c.k, int(c.largest), c.alpha, c.beta, p.flags,
            self.theta.data_ptr() if self.exchange_theta else None, self.s_val.data_ptr(), self.s_idx.data_ptr(),
            self.index_offset, p.ws.data_ptr(), p.ws_bytes, s.cuda_stream, None), "dtopk_select_finish")
        self.send[0:1].copy_(self.kout)

    def step(self, keys: torch.Tensor | None = None) -> None:
        """One sharded top-k; results in ``self.values`` / ``self.indices`` (stream-ordered)."""
        if self.graph is not None and keys is None:
            self.graph.replay()
            return
        from . import _native

        s = torch.cuda.current_stream(self.device)
        if self.local is not None:
            self._local(self.dv.keys if keys is None else keys, s)
        elif self.exchange_theta:  # empty shard: joins the exchange with theta = 0, sends no pairs
            self.theta.zero_()
            dist.all_reduce(self.theta, op=dist.ReduceOp.MAX, group=self.group)
        lib, w, kl = self.lib, self.world, self.kl
        largest = int(self.largest)
        if self.merge_mode == "gather":
            _all_gather_flat(self.gathered, self.send, self.group)
            g = self.gathered
            _native.check(lib.dtopk_merge_lists(
                self.code, largest, g.data_ptr() + 8 * (2 + kl), 2, 1, g.data_ptr() + 16, None, self.pw, g.data_ptr(),
                self.pw, w, self.k, self.values.data_ptr(), self.indices.data_ptr(), self.tmp_val.data_ptr(),
                self.tmp_idx.data_ptr(), self.tmp_len.data_ptr(), s.cuda_stream), "dtopk_merge_lists")
            return
        self._select_merge(s)

    def _select_merge(self, s) -> None:
        """Distributed radix select + exact-k assembly (class docstring)."""
        from . import _native

        lib, cs = self.lib, s.cuda_stream
        cnt = self.send.data_ptr()
        bits = self.s_val.data_ptr()
        largest = int(self.largest)
        _native.check(lib.dtopk_dsel_init(self.state.data_ptr(), self.hist.data_ptr(), self.k, cs), "dsel_init")
        for pas in range(3):
            _native.check(lib.dtopk_dsel_hist(self.code, largest, bits, cnt, self.kl, self.state.data_ptr(), pas,
                                              self.hist.data_ptr(), cs), "dsel_hist")
            dist.all_reduce(self.hist, op=dist.ReduceOp.SUM, group=self.group)
            _native.check(lib.dtopk_dsel_digit(self.code, largest, self.state.data_ptr(), self.hist.data_ptr(), pas,
                                               bits, cnt, self.gt_eq.data_ptr(), cs), "dsel_digit")
        _all_gather_flat(self.g_cnt, self.gt_eq, self.group)
        w, k = self.world, self.k
        _native.check(lib.dtopk_dsel_place(self.g_cnt.data_ptr(), self.state.data_ptr(), self.rank, w, k, bits,
                                           self.s_idx.data_ptr(), self.slots.data_ptr(), self.seg.data_ptr(),
                                           self.seg.data_ptr() + 8 * w, cs), "dsel_place")
        dist.all_reduce(self.slots, op=dist.ReduceOp.SUM, group=self.group)
        sl = self.slots
        _native.check(lib.dtopk_merge_lists(
            self.code, largest, sl.data_ptr(), 2, 2, sl.data_ptr() + 8 * k, self.seg.data_ptr(), 0,
            self.seg.data_ptr() + 8 * w, 1, w, k, self.values.data_ptr(), self.indices.data_ptr(),
            self.tmp_val.data_ptr(), self.tmp_idx.data_ptr(), self.tmp_len.data_ptr(), cs), "dtopk_merge_lists")

    def capture(self, warmup: int = 2) -> None:
        """Capture one whole step (kernels + NCCL collectives) in a CUDA graph;
        later ``step()`` calls (without new keys) replay it."""
        if dist.get_backend(self.group) != "nccl":
            raise RuntimeError("graph capture of the sharded step needs the NCCL backend")
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.step()
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self.step()
        torch.cuda.synchronize(self.device)
        self.graph = g

    def result(self) -> TopKResult:
        """Synchronise and wrap the last step's answer."""
        from . import _native

        stats = WorkloadStats()
        if self.merge_mode == "gather":
            pairs = int(self.gathered.view(self.world, self.pw)[:, 0].sum().item())
        else:
            pairs = self.k
        stats.device = {"merge": self.merge_mode, "gathered_pairs": pairs, "theta_global": int(self.theta.item())}
        last = self.values[-1:]
        thr = float(last.item()) if self.code == _native.DTYPE_F32 else int(last.view(torch.int32).item()) & 0xFFFFFFFF
        return TopKResult(values=self.values, threshold=thr, stats=stats, indices=self.indices)


_SEL_BINS = 2048
_SEL_DIGITS = ((21, 11), (10, 11), (0, 10))  # (shift, bits) of the 32-bit order key, most significant first


def select_contribution(key: torch.Tensor, cnt: torch.Tensor, k: int, rank: int, group,
                        hist: torch.Tensor | None = None, g_cnt: torch.Tensor | None = None):
    """Distributed radix select over per-rank candidate lists (ShardedTopK merge="select").

    ``key``: this rank's candidates' int64 order keys (larger = better), the
    first ``cnt`` (int64[1] tensor) of them valid and ordered (key desc, index
    asc); the union over ranks holds the global top-k.  Returns (mine, pre),
    int64[1] tensors: this rank contributes its first ``mine`` candidates at
    offset ``pre`` of the k-slot answer.  Ranks are in global index order, so
    kth-key ties are granted to lower ranks first.  No host synchronisation.
    """
    dev = key.device
    hist = torch.empty(_SEL_BINS, dtype=torch.int64, device=dev) if hist is None else hist
    world = dist.get_world_size(group)
    g_cnt = torch.empty(2 * world, dtype=torch.int64, device=dev) if g_cnt is None else g_cnt
    zero1 = torch.zeros(1, dtype=torch.int64, device=dev)
    valid = torch.arange(key.numel(), device=dev) < cnt
    prefix = zero1.clone()
    rem = torch.full_like(zero1, k)
    for shift, nb in _SEL_DIGITS:
        digit = (key >> shift) & ((1 << nb) - 1)
        match = valid & ((key >> (shift + nb)) == prefix)
        hist.zero_().scatter_add_(0, digit, match.to(torch.int64))
        dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
        # at_least[d] = #candidates (all ranks) under this prefix with digit >= d
        at_least = torch.cat([hist.flip(0).cumsum(0).flip(0), zero1])
        d = (at_least[:-1] >= rem).sum(0, keepdim=True) - 1
        rem = rem - at_least.index_select(0, d + 1)
        prefix = (prefix << nb) | d
    kth = prefix
    gt = (valid & (key > kth)).sum(0, keepdim=True)
    eq = (valid & (key == kth)).sum(0, keepdim=True)
    _all_gather_flat(g_cnt, torch.cat([gt, eq]), group)
    g = g_cnt.view(-1, 2)
    eq_before = torch.cumsum(g[:, 1], 0) - g[:, 1]
    take = torch.minimum(torch.clamp(rem - eq_before, min=0), g[:, 1])
    contrib = g[:, 0] + take
    pre = torch.cumsum(contrib, 0) - contrib
    return contrib[rank:rank + 1], pre[rank:rank + 1]


def _order_key(bits: torch.Tensor, code: int, largest: bool) -> torch.Tensor:
    """int32 raw bits of u32/f32 values -> int64 order key in [0, 2^32), larger = better."""
    from . import _native

    kk = bits.to(torch.int64) & 0xFFFFFFFF
    if code == _native.DTYPE_F32:
        kk = torch.where(kk >> 31 == 1, kk ^ 0xFFFFFFFF, kk | 0x80000000)
    if not largest:
        kk = 0xFFFFFFFF - kk
    return kk


def _all_gather_flat(out: torch.Tensor, inp: torch.Tensor, group) -> None:
    """all_gather of equal-size contributions into one flat tensor (rank order)."""
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)
    else:  # gloo (CPU tests, or several ranks sharing one GPU): list form
        dist.all_gather(list(out.chunk(dist.get_world_size(group))), inp, group=group)


def _dev_of(x):
    return x.device if isinstance(x, torch.Tensor) else torch.device("cpu")


def _as_gatherable(ts):
    # NCCL/gloo lack uint32 all_gather: move the bits as int32
    return [t.view(torch.int32) if t.dtype == torch.uint32 else t for t in ts]


# ---------------------------------------------------------------------------
# Partitioned run on one GPU with streamed partitions (reference:
# distributed.run_distributed, distributed.py:140-251)
# ---------------------------------------------------------------------------
@dataclass
class GatherMessage:
    """One worker's contribution (distributed.py:63-75): its local top-k
    (device tensors, values best first plus global indices) and lane timings."""

    worker_id: int
    local_topk: torch.Tensor
    local_indices: torch.Tensor
    compute_nanos: int
    reload_nanos: int
    sent_at_nanos: int = 0

    def payload_bytes(self) -> int:
        return (self.local_topk.element_size() + 8) * int(self.local_topk.numel())


@dataclass
class DistributedReport:
    result: TopKResult
    messages: list
    received_at_nanos: list
    gathered_bytes: int
    total_nanos: int
    reloaded_partitions: int = 0
    extra: dict = field(default_factory=dict)

    def communication_nanos(self, worker_id: int) -> int:
        msg = self.messages[worker_id]
        return max(0, self.received_at_nanos[worker_id] - msg.sent_at_nanos)


def _merge_by_index(values: torch.Tensor, indices: torch.Tensor, k: int, largest: bool):
    """Exact top-k of (value, global index) pairs under (value best first,
    index ascending): order the pairs by index, then the device top-k's
    position tie-break is the index tie-break."""
    from .pipeline import dr_topk

    order = torch.argsort(indices)
    # torch has no uint32 gather on CUDA: move the bits as int32
    bits = values.view(torch.int32) if values.dtype == torch.uint32 else values
    v, i = bits[order], indices[order]
    if values.dtype == torch.uint32:
        v = v.view(torch.uint32)
    r = dr_topk(v, PipelineConfig(k=min(k, v.numel()), alpha=0, auto_alpha=False, largest=largest))
    return r.values, i[r.indices]


def _worker_lane(worker_id, source, parts, plan_, k, cfg, device, outbox):
    from ._device import to_device
    from .data import read_vector
    from .pipeline import dr_topk

    try:
        torch.cuda.set_device(device)
        stream = torch.cuda.Stream(device)
        with torch.cuda.stream(stream):
            is_file = not isinstance(source, (np.ndarray, torch.Tensor))
            stage, stage_ev = None, [None, None]
            copy = torch.cuda.Stream(device)
            if is_file:
                cap = max(plan_.partitions[i].length for i in parts) if parts else 1
                # two pinned staging buffers: the file read of one partition overlaps
                # the H2D of the previous one (copy stream) and the top-k before it
                stage = [torch.empty(cap, dtype=torch.uint32, pin_memory=True) for _ in range(2)]

            def load(part, slot=0):
                if not is_file:
                    chunk = source[part.offset:part.offset + part.length]
                    return to_device(chunk, device).keys if not isinstance(chunk, torch.Tensor) or not chunk.is_cuda \
                        else chunk
                if stage_ev[slot] is not None:
                    stage_ev[slot].synchronize()  # its previous H2D has finished reading it
                buf = stage[slot]
                read_vector(source, offset=part.offset, count=part.length, out=buf.numpy()[: part.length])
                dev = torch.empty(part.length, dtype=torch.uint32, device=device)
                copy.wait_stream(stream)
                with torch.cuda.stream(copy):
                    dev.copy_(buf[: part.length], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(copy)
                stage_ev[slot] = ev
                stream.wait_event(ev)  # the top-k of this partition runs after its copy
                dev.record_stream(stream)
                return dev

            resident = {i: load(plan_.partitions[i]) for i in parts if plan_.partitions[i].resident}
            reload_nanos, vals, idxs = 0, [], []
            t_compute = time.perf_counter_ns()
            streamed = [i for i in parts if i not in resident]
            prefetched = {}
            if streamed:  # the first reload starts before any compute
                t0 = time.perf_counter_ns()
                prefetched[streamed[0]] = load(plan_.partitions[streamed[0]], 0)
                reload_nanos += time.perf_counter_ns() - t0
            for i in parts:
                part = plan_.partitions[i]
                if i in resident:
                    chunk = resident.pop(i)
                else:  # a partition beyond the residency cap: streamed from the file (reload overhead)
                    chunk = prefetched.pop(i)
                    pos = streamed.index(i)
                    if pos + 1 < len(streamed):  # read the next one while this one is on the GPU
                        t0 = time.perf_counter_ns()
                        nxt = streamed[pos + 1]
                        prefetched[nxt] = load(plan_.partitions[nxt], (pos + 1) % 2)
                        reload_nanos += time.perf_counter_ns() - t0
                r = dr_topk(chunk, replace(cfg, k=min(k, part.length)))
                vals.append(r.values)
                idxs.append(r.indices + part.offset)
                del chunk
            if vals:
                v, ix = torch.cat(vals), torch.cat(idxs)
                if len(vals) > 1:
                    v, ix = _merge_by_index(v, ix, k, cfg.largest)
            else:  # more workers than partitions: this lane owns nothing
                v = torch.empty(0, dtype=torch.uint32, device=device)
                ix = torch.empty(0, dtype=torch.int64, device=device)
            stream.synchronize()
            compute_nanos = time.perf_counter_ns() - t_compute - reload_nanos
        msg = GatherMessage(worker_id, v, ix, compute_nanos, reload_nanos)
        msg.sent_at_nanos = time.perf_counter_ns()
        outbox.put((worker_id, msg, None))
    except BaseException as exc:  # surfaced as WorkerFailed by the coordinator
        outbox.put((worker_id, None, exc))


def run_distributed(source, k: int, cfg: PipelineConfig | None = None, workers: int = 1, *,
                    max_resident: int = DEFAULT_MAX_RESIDENT, device=None) -> DistributedReport:
    """Partitioned top-k with gather-to-primary aggregation on the GPU.

    ``source``: a numpy / torch vector or a DTKV file path.  The partition
    plan is the reference's (``plan``); worker lanes are threads with their
    own CUDA streams.  Partitions beyond a worker's first are streamed from
    the file (pinned staging, H2D) when the residency cap forces it -- the
    out-of-HBM path -- and their read time is reported as reload overhead.
    Every lane sends its local top-k with global indices; the coordinator
    merges them exactly (value best first, lowest index on ties).
    """
    from ._device import to_caller
    from .data import read_header

    start = time.perf_counter_ns()
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if isinstance(source, (str, bytes)) or hasattr(source, "__fspath__"):
        n, kind = read_header(source), "numpy"
    elif isinstance(source, torch.Tensor):
        n, kind = int(source.numel()), ("torch_cuda" if source.is_cuda else "torch_cpu")
    else:
        source = np.ascontiguousarray(np.asarray(source)).ravel()
        if source.dtype != np.float32:
            source = source.astype(np.uint32)
        n, kind = source.size, "numpy"
    cfg = cfg if cfg is not None else PipelineConfig(k=k)
    plan_ = plan(n, k, workers, max_resident)
    outbox: queue.Queue = queue.Queue()
    lanes = [threading.Thread(target=_worker_lane, args=(w, source, plan_.assignments[w], plan_, k, cfg, device,
                                                         outbox), name=f"dtopk-worker-{w}", daemon=True)
             for w in range(workers)]
    for t in lanes:
        t.start()
    messages, received, failure = [None] * workers, [0] * workers, None
    for _ in range(workers):
        wid, msg, exc = outbox.get()
        received[wid] = time.perf_counter_ns()
        if exc is not None and failure is None:
            failure = (wid, exc)
        messages[wid] = msg
    for t in lanes:
        t.join()
    if failure is not None:
        raise WorkerFailed(f"worker {failure[0]} failed: {failure[1]!r}") from failure[1]
    v = torch.cat([m.local_topk.to(device) for m in messages])
    ix = torch.cat([m.local_indices.to(device) for m in messages])
    fv, fi = _merge_by_index(v, ix, k, cfg.largest)
    torch.cuda.synchronize(device)
    stats = WorkloadStats()
    res = TopKResult(values=to_caller(fv, kind), threshold=to_caller(fv[-1:], "numpy")[0].item(), stats=stats, indices=to_caller(fi, kind))
    reloaded = sum(1 for w, ps in plan_.assignments.items() for i in ps if not plan_.partitions[i].resident)
    return DistributedReport(result=res, messages=messages, received_at_nanos=received,
                             gathered_bytes=sum(m.payload_bytes() for m in messages),
                             total_nanos=time.perf_counter_ns() - start, reloaded_partitions=reloaded)
