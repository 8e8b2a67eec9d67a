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
for dist_name, n_local, k, largest in [("uniform", 1 << 22, 1000, True), ("uniform", (1 << 22) + 37, 70000, True),
                                       ("few_distinct", 1 << 21, 5000, True), ("all_equal", 1 << 21, 3000, False),
                                       ("normal_f32", 1 << 22, 4096, True), ("uniform", 1 << 20, 1 << 19, True),
                                       ("all_equal", 1 << 20, 1 << 18, True), ("few_distinct", 1 << 20, 300001, False),
                                       ("normal_f32", (1 << 20) + 5, 1 << 17, False)]:
    n_total = n_local * world
    full = data.generate(dist_name, n_total, seed=7, device=dev)
    lo, ln = dtopk.shard_bounds(n_total, world, rank)
    shard = full[lo:lo + ln].clone()
    cfg = dtopk.PipelineConfig(k=k, largest=largest)
    st = dtopk.ShardedTopK(shard, n_total, k, cfg)
    for _ in range(2):
        st.step()
    r = st.result()
    other = "select" if st.merge_mode == "gather" else "gather"
    st3 = dtopk.ShardedTopK(shard, n_total, k, cfg, merge=other)
    for _ in range(2):
        st3.step()
    r3 = st3.result()
    r2 = dtopk.sharded_topk(shard, n_total, k, cfg)
    torch.cuda.synchronize()
    if rank == 0:
        from oracle import oracle

        host = full.cpu().numpy()
        keys = oracle.to_keys(host, largest)
        ek, ei = oracle.topk_with_indices(keys, k)
        for name, res in ((f"ShardedTopK/{st.merge_mode}", r), (f"ShardedTopK/{other}", r3),
                          ("sharded_topk", r2)):
            gi = res.indices.cpu().numpy()
            gv = res.values.cpu().numpy()
            good = np.array_equal(gi, ei) and np.array_equal(oracle.to_keys(gv, largest), ek)
            ok &= good
            print(f"{name:20s} {dist_name:12s} world={world} n_local={n_local} k={k} largest={largest}: "
                  f"{'OK' if good else 'MISMATCH'}", flush=True)
dist.barrier()
dist.destroy_process_group()
if rank == 0:
    print("ALL OK" if ok else "FAILURES")
    sys.exit(0 if ok else 1)
