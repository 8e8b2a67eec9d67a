"""Row f3: alpha sweep of the GPU pipeline (reference CSV schema) and the B200 const of Eq. 11.

    python tools/alpha_sweep.py [--log2n 30] [--out gpurun_out/alpha_sweep.csv]

For every k, alphas auto-2 .. auto+3 (const 3) go through tuning.sweep (stage
times from CUDA events, values verified against a device sort) and through a
CUDA-graph replay timing; the alpha with the lowest replay time is the
measured optimum, and tuning.b200_const fits Eq. 11's const to those optima.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2109_08219_b200 as dtopk  # noqa: E402
from paper_2109_08219_b200 import _native, data, tuning  # noqa: E402
from paper_2109_08219_b200.pipeline import DrTopK  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2n", type=int, default=30)
ap.add_argument("--ks", default="1,32,1024,8192,65536,262144,1048576")
ap.add_argument("--out", default="gpurun_out/alpha_sweep.csv")
args = ap.parse_args()
n = 1 << args.log2n
v = data.generate("uniform", n, seed=3, device="cuda")
s = torch.cuda.current_stream()
rows, best, report = [], {}, []
for k in [int(x) for x in args.ks.split(",")]:
    a0 = tuning.auto_alpha(n, k)
    alphas = [a for a in range(a0 - 2, a0 + 4) if a >= 1 and 2 * (n >> a) >= k]
    rows += tuning.sweep(v, k, alphas=alphas, repeats=5, verify=True)
    # plans first, then interleaved rounds: run-order drift (clocks, HBM temperature) hits every alpha alike
    plans = {a: DrTopK(n, dtopk.PipelineConfig(k=k, alpha=a, auto_alpha=False), _native.DTYPE_U32, torch.uint32,
                       v.device, timed=False, use_graph=True) for a in alphas}
    for p in plans.values():
        for _ in range(3):
            p.launch(v, s)
    g = {a: [] for a in alphas}
    for _ in range(7):
        for a, p in plans.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(10):
                p.launch(v, s)
            e1.record(s)
            torch.cuda.synchronize()
            g[a].append(e0.elapsed_time(e1) / 10)
    times = {a: round(statistics.median(x), 4) for a, x in g.items()}
    del plans
    a_best = min(times, key=times.get)
    best[(n, k)] = a_best
    report.append({"k": k, "auto_alpha_const3": a0, "best_alpha": a_best, "graph_ms": times})
    print(json.dumps(report[-1]), flush=True)
os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
tuning.write_csv(rows, args.out)
c = tuning.b200_const(best)
print(json.dumps({"b200_const": round(c, 3), "auto_alpha_b200": {k: tuning.auto_alpha(n, k, c) for (_, k) in best}}))
