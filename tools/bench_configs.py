"""Time BASELINE configs 3-5 (float32 / adversarial / 2^33) on one GPU.

    python tools/bench_configs.py [--steps 20] [--only adversarial|float|big]

Same method as bench.py: CUDA-graph plans, inputs resident in HBM (>> L2),
CUDA events around back-to-back steps.  Prints one JSON object per case.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2109_08219_b200 as dtopk  # noqa: E402
from paper_2109_08219_b200 import _native, data  # noqa: E402
from paper_2109_08219_b200.pipeline import DrTopK  # noqa: E402


def run_case(name, v, k, steps, beta=2, largest=True, log2n=30):
    n = v.numel()
    code = _native.DTYPE_F32 if v.dtype == torch.float32 else _native.DTYPE_U32
    p = DrTopK(n, dtopk.PipelineConfig(k=k, beta=beta, largest=largest), code, v.dtype, v.device, timed=False,
               use_graph=True)
    s = torch.cuda.current_stream()
    for _ in range(3):
        p.launch(v, s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(steps):
        p.launch(v, s)
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    h = p.header()
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
    out = {"case": name, "n": n, "k": k, "beta": p.cfg.beta, "alpha": p.cfg.alpha, "ms": round(ms, 4),
           "keys_per_s": n / (ms * 1e-3), "frac_of_peak": n * 4 / (ms * 1e-3) / 1e9 / peak,
           "path": int(h.path), "pool_gt": int(h.pool_gt), "candidates": int(h.candidate_subranges),
           "reread": int(h.elements_reread), "fq": int(h.fully_qualified), "pq": int(h.partially_qualified)}
    print(json.dumps(out), flush=True)
    del p
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--only", default="all")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = 1 << 30
    if args.only in ("all", "float"):
        for dist in ("normal_f32", "pareto_f32"):
            v = data.generate(dist, n, seed=1, device=dev)
            for beta in (1, 2, 3):
                run_case(f"config3 {dist} beta={beta}", v, 1024, args.steps, beta=beta)
            del v
    if args.only in ("all", "adversarial"):
        for dist in ("ascending", "all_equal", "few_distinct", "nd_u32"):
            v = data.generate(dist, n, seed=1, device=dev)
            run_case(f"config4 {dist}", v, 1 << 16, args.steps)
            del v
    if args.only in ("big",):
        v = data.generate("uniform", 1 << 33, seed=1, device=dev)
        for k in (1 << 10, 1 << 20):
            run_case("config5 2^33 single GPU", v, k, max(3, args.steps // 4), log2n=33)


if __name__ == "__main__":
    main()
