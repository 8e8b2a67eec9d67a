"""CPU: the multi-rank exchange / merge logic of sharded_topk on gloo (world size 2).

The per-rank compute is the oracle (test stand-in for the GPU pipeline):
delegates -> theta_r = kth(D_r) -> all_reduce(MAX) -> elements >= theta* of the
shard, (key desc, index asc) -> all_gather -> exact merge.  The product runs
the same orchestration with ``DeviceOps`` (libdtopk.so) over NCCL.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class OracleOps:
    """Host stand-in for DeviceOps (tests only)."""

    def __init__(self, oracle_mod):
        self.o = oracle_mod

    def begin(self, shard, cfg):
        keys = shard.numpy().view(np.uint32)
        if cfg.direct_fallback:
            return (keys, cfg), None
        d = self.o.extract_delegates(keys, cfg.alpha, cfg.beta)
        theta = self.o.radix_threshold(d, cfg.k, False)
        return (keys, cfg), torch.tensor([theta], dtype=torch.int64)

    def finish(self, state, theta, index_offset):
        keys, cfg = state
        th = int(theta.item()) if theta is not None else 0
        idx = np.flatnonzero(keys >= np.uint32(th))
        order = np.lexsort((idx, ~keys[idx]))[: cfg.k]
        sel = idx[order]
        return torch.from_numpy(keys[sel].astype(np.uint32)), torch.from_numpy(sel.astype(np.int64) + index_offset)

    def merge(self, values, indices, k, largest):
        v = values.numpy().view(np.uint32) if values.dtype != torch.uint32 else values.numpy()
        order = np.lexsort((np.arange(v.size), ~v))[:k]
        return torch.from_numpy(v[order]), indices[torch.from_numpy(order)]


def _worker(rank, world, port, n, k, seed, exchange, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import oracle

        import paper_2109_08219_b200 as dtopk

        v = oracle.generate_uniform(n, seed=seed) if seed >= 0 else np.arange(n, dtype=np.uint32) % 97
        lo, ln = dtopk.shard_bounds(n, world, rank)
        shard = torch.from_numpy(v[lo:lo + ln].copy())
        r = dtopk.sharded_topk(shard, n, k, exchange_theta=exchange, ops=OracleOps(oracle))
        out[rank] = (r.values.numpy().astype(np.uint32), r.indices.numpy(), r.stats.device)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("exchange", [True, False])
@pytest.mark.parametrize("seed,k", [(5, 300), (6, 1), (-1, 500)])
def test_sharded_topk_gloo_world2(exchange, seed, k, oracle_mod):
    n, world = 40_000, 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, n, k, seed, exchange, out), nprocs=world, join=True,
                       start_method="spawn")
    v = oracle_mod.generate_uniform(n, seed=seed) if seed >= 0 else np.arange(n, dtype=np.uint32) % 97
    ek, ei = oracle_mod.topk_with_indices(v, k)
    for r in range(world):
        vals, idx, dev = out[r]
        np.testing.assert_array_equal(idx, ei)
        np.testing.assert_array_equal(vals, ek)
        assert dev["gathered_pairs"] <= world * k
    # the theta exchange can only shrink what is gathered
    if exchange:
        assert out[0][2]["theta_global"] >= 0


def _select_worker(rank, world, port, n, k, seed, out):
    """ShardedTopK merge="select" arithmetic on CPU tensors: per-rank candidate
    lists (shard top-k, garbage past the count) -> select_contribution ->
    all_reduce assembly of exactly k pairs -> stable order."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import oracle

        import paper_2109_08219_b200 as dtopk
        from paper_2109_08219_b200.distributed import select_contribution

        v = oracle.generate_uniform(n, seed=seed) if seed >= 0 else (np.arange(n, dtype=np.uint32) % 13) << 28
        lo, ln = dtopk.shard_bounds(n, world, rank)
        sh = v[lo:lo + ln]
        kl = min(k, ln)
        # odd ranks hold fewer than kl valid pairs (a theta* cut): never below what the global top-k needs here
        _, gi = oracle.topk_with_indices(v, k)
        need = int(((gi >= lo) & (gi < lo + ln)).sum())
        cnt = max(need, kl - (rank % 2))
        order = np.lexsort((np.arange(ln), ~sh))[:cnt]
        key = np.full(kl, 0xFFFFFFFF, dtype=np.int64)  # garbage past cnt must be ignored
        key[:cnt] = sh[order]
        idx = np.full(kl, -7, dtype=np.int64)
        idx[:cnt] = order + lo
        key_t, idx_t = torch.from_numpy(key), torch.from_numpy(idx)
        mine, pre = select_contribution(key_t, torch.tensor([cnt]), k, rank, None)
        j = torch.arange(kl)
        dest = torch.where(j < mine, pre + j, torch.full_like(j, k))
        vals = torch.zeros(k + 1, dtype=torch.int64).scatter_(0, dest, key_t)
        ids = torch.zeros(k + 1, dtype=torch.int64).scatter_(0, dest, idx_t)
        dist.all_reduce(vals)
        dist.all_reduce(ids)
        vals, ids = vals[:k], ids[:k]
        o = torch.sort(vals, descending=True, stable=True).indices
        out[rank] = (vals[o].numpy().astype(np.uint32), ids[o].numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("seed,k", [(8, 5000), (9, 1), (-1, 4000)])
def test_select_merge_gloo(world, seed, k, oracle_mod):
    n = 30_011
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_select_worker, args=(world, port, n, k, seed, out), nprocs=world, join=True,
                       start_method="spawn")
    v = oracle_mod.generate_uniform(n, seed=seed) if seed >= 0 else (np.arange(n, dtype=np.uint32) % 13) << 28
    ek, ei = oracle_mod.topk_with_indices(v, k)
    for r in range(world):
        vals, idx = out[r]
        np.testing.assert_array_equal(idx, ei)
        np.testing.assert_array_equal(vals, ek)


class FailingOps(OracleOps):
    """Rank 1 fails in begin (e.g. an out-of-memory or a bad shard)."""

    def begin(self, shard, cfg):
        if dist.get_rank() == 1:
            raise RuntimeError("injected failure")
        return super().begin(shard, cfg)


def _edge_worker(rank, world, port, n, k, fail, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import oracle

        import paper_2109_08219_b200 as dtopk

        v = oracle.generate_uniform(n, seed=11)
        lo, ln = dtopk.shard_bounds(n, world, rank)
        shard = torch.from_numpy(v[lo:lo + ln].copy())
        ops = FailingOps(oracle) if fail else OracleOps(oracle)
        try:
            r = dtopk.sharded_topk(shard, n, k, ops=ops)
            out[rank] = ("ok", r.values.numpy().astype(np.uint32), r.indices.numpy())
        except Exception as exc:  # noqa: BLE001 -- the test inspects the type
            out[rank] = (type(exc).__name__, None, None)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,k", [
    (2, 1, 1),                 # rank 1's shard is empty
    (3, 3 * 1000 + 1, 1500),   # ragged last shard, k above every shard's length
    (3, 2, 2),                 # an empty shard and one-key shards (direct path)
    (2, 20_001, 9_000),        # k close to a shard's length
])
def test_sharded_topk_ragged_and_empty_shards(world, n, k, oracle_mod):
    """Every rank joins every collective whatever its shard (ragged
    last shards and empty shards must not desynchronise the collectives)."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_edge_worker, args=(world, _free_port(), n, k, False, out), nprocs=world, join=True,
                       start_method="spawn")
    v = oracle_mod.generate_uniform(n, seed=11)
    ek, ei = oracle_mod.topk_with_indices(v, k)
    for r in range(world):
        status, vals, idx = out[r]
        assert status == "ok"
        np.testing.assert_array_equal(idx, ei)
        np.testing.assert_array_equal(vals, ek)


def test_sharded_topk_failure_reaches_every_rank(oracle_mod):
    """A rank that fails in begin raises WorkerFailed on every rank instead of
    leaving its peers blocked in the theta all-reduce (distributed.py:238-241)."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_edge_worker, args=(2, _free_port(), 50_000, 100, True, out), nprocs=2, join=True,
                       start_method="spawn")
    assert out[0][0] == "WorkerFailed" and out[1][0] == "WorkerFailed"
