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
