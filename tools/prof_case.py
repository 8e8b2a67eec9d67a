"""One eager dr_topk per call on a chosen input, for ncu launch lists / captures.

    python tools/prof_case.py --dist ascending --k 65536 [--log2n 30] [--reps 4]

The input is generated on the device (same generators as the tests); the call
is repeated --reps times so `ncu -s/-c` can skip the warm-up launches.
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2109_08219_b200 as dtopk  # noqa: E402
from paper_2109_08219_b200 import data  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dist", default="uniform")
    ap.add_argument("--k", type=int, default=1024)
    ap.add_argument("--log2n", type=int, default=30)
    ap.add_argument("--beta", type=int, default=2)
    ap.add_argument("--smallest", action="store_true")
    ap.add_argument("--reps", type=int, default=4)
    a = ap.parse_args()
    v = data.generate(a.dist, 1 << a.log2n, seed=2, device="cuda")
    cfg = dtopk.PipelineConfig(k=a.k, beta=a.beta, largest=not a.smallest)
    for _ in range(a.reps):
        r = dtopk.dr_topk(v, cfg)
    torch.cuda.synchronize()
    print(a.dist, a.k, r.stats.device)


if __name__ == "__main__":
    main()
