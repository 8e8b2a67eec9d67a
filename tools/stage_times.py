"""Median per-stage device times (CUDA events on the launch stream) over many
eager steps, plus the median graph-replay step, for a list of k.

    DTOPK_LIB=... python tools/stage_times.py [--log2n 30] [--reps 30] [--ks 1,1024,...]

Post-K1 stages do not depend on K1's run-to-run HBM variance, so this is the
A/B tool for the FirstK / Concat / SecondK kernels.
"""
import argparse
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2109_08219_b200 as dtopk  # noqa: E402
from paper_2109_08219_b200 import _native, data  # noqa: E402
from paper_2109_08219_b200.pipeline import DrTopK  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2n", type=int, default=30)
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--ks", default="1,16,256,1024,4096,16384,65536,262144,1048576")
ap.add_argument("--dist", default="uniform")
ap.add_argument("--alphas", default="", help="comma list of manual alphas per k (auto if empty)")
ap.add_argument("--const", type=float, default=3.0, help="auto_alpha const_c")
ap.add_argument("--beta", type=int, default=2)
args = ap.parse_args()
lib = _native.load()
n = 1 << args.log2n
v = data.generate(args.dist, n, seed=1000, device="cuda")
s = torch.cuda.current_stream()
ev = [[lib.dtopk_event_create() for _ in range(5)] for _ in range(args.reps)]
arr = [(ctypes.c_void_p * 5)(*e) for e in ev]
out = {}
ks = [int(x) for x in args.ks.split(",")]
alphas = [int(x) for x in args.alphas.split(",")] if args.alphas else [None] * len(ks)
for k, al in zip(ks, alphas):
    cfg = (dtopk.PipelineConfig(k=k, const_c=args.const, beta=args.beta) if al is None
           else dtopk.PipelineConfig(k=k, alpha=al, auto_alpha=False, beta=args.beta))
    p = DrTopK(n, cfg, _native.DTYPE_U32, torch.uint32, v.device, timed=False, use_graph=True)
    for _ in range(3):
        p.launch(v, s)
    for i in range(args.reps):
        p.launch(v, s, events=arr[i])
    torch.cuda.synchronize()
    st = {name: statistics.median(lib.dtopk_event_elapsed_ms(e[j], e[j + 1]) for e in ev)
          for j, name in enumerate(dtopk.STAGES)}
    st["post_k1"] = statistics.median(lib.dtopk_event_elapsed_ms(e[1], e[4]) for e in ev)
    g = []
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        a.record(s)
        for _ in range(10):
            p.launch(v, s)
        b.record(s)
        torch.cuda.synchronize()
        g.append(a.elapsed_time(b) / 10)
    st["graph_step"] = statistics.median(g)
    out[k] = {x: round(y * 1000, 1) for x, y in st.items()}  # microseconds
    h = p.header()
    print(k, "alpha", p.cfg.alpha, out[k], "pool_gt", int(h.pool_gt), "reread", int(h.elements_reread), "path", int(h.path), flush=True)
    del p
