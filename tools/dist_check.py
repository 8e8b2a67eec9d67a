"""Multi-rank check of the sharded path on GPU (tooling; oracle is the checker).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/dist_check.py

DTOPK_DIST_BACKEND=gloo lets several ranks share one GPU (NCCL refuses
duplicate devices), which is how the exchange/merge runs on a 1-GPU box.
Compares ShardedTopK and sharded_topk with the oracle on the full vector.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2109_08219_b200 as dtopk  # noqa: E402
from paper_2109_08219_b200 import data  # noqa: E402

backend = os.environ.get("DTOPK_DIST_BACKEND", "nccl")
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
dev = torch.device("cuda", local % torch.cuda.device_count())
torch.cuda.set_device(dev)
dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
ok = True
# (distribution, n_total, k, largest): n_total need not divide by world (ragged last
# shard, shards shorter than k, an empty shard when n_total < world)
CASES = [("uniform", (1 << 22) * world, 1000, True), ("uniform", ((1 << 22) + 37) * world, 70000, True),
         ("few_distinct", (1 << 21) * world, 5000, True), ("all_equal", (1 << 21) * world, 3000, False),
         ("normal_f32", (1 << 22) * world, 4096, True), ("uniform", (1 << 20) * world, 1 << 19, True),
         ("all_equal", (1 << 20) * world, 1 << 18, True), ("few_distinct", (1 << 20) * world, 300001, False),
         ("normal_f32", ((1 << 20) + 5) * world, 1 << 17, False),
         ("uniform", 4 * 100003 * world + 1, 100003 * world + 1, True),   # ragged: k above the short shard
         ("uniform", 4 * 100003 * world + 1, 150000, True),
         ("uniform", world - 1 if world > 1 else 1, 1, True),              # an empty shard
         ("uniform", 5000 * world + 3, 7, False)]                          # tiny shards: direct path
for dist_name, n_total, k, largest in CASES:
    full = data.generate(dist_name, n_total, seed=7, device=dev)
    lo, ln = dtopk.shard_bounds(n_total, world, rank)
    shard = full[lo:lo + ln].clone()
    cfg = dtopk.PipelineConfig(k=k, largest=largest)
    runs = []
    for merge in ("gather", "select"):
        for exch in (True, False):
            st = dtopk.ShardedTopK(shard, n_total, k, cfg, merge=merge, exchange_theta=exch)
            for _ in range(2):
                st.step()
            r = st.result()
            runs.append((f"ShardedTopK/{merge}/x{int(exch)}", (r.values.clone(), r.indices.clone())))
            if backend == "nccl" and exch:
                st.capture()
                st.step()
                r = st.result()
                runs.append((f"ShardedTopK/{merge}/graph", (r.values.clone(), r.indices.clone())))
    r = dtopk.sharded_topk(shard, n_total, k, cfg)
    runs.append(("sharded_topk", (r.values, r.indices)))
    torch.cuda.synchronize()
    if rank == 0:
        from oracle import oracle

        host = full.cpu().numpy()
        keys = oracle.to_keys(host, largest)
        ek, ei = oracle.topk_with_indices(keys, k)
        for name, (rv, ri) in runs:
            gi = ri.cpu().numpy()
            gv = rv.cpu().numpy()
            good = np.array_equal(gi, ei) and np.array_equal(oracle.to_keys(gv, largest), ek)
            ok &= good
            print(f"{name:24s} {dist_name:12s} world={world} n_total={n_total} k={k} largest={largest}: "
                  f"{'OK' if good else 'MISMATCH'}", flush=True)
dist.barrier()
dist.destroy_process_group()
if rank == 0:
    print("ALL OK" if ok else "FAILURES")
    sys.exit(0 if ok else 1)
