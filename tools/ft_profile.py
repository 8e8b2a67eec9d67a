"""Phase clocks of fast_tail (library built with -DDTOPK_FT_PROFILE, via DTOPK_LIB).

    DTOPK_LIB=paper_2109_08219_b200/_lib/var/lib_ftprof.so python tools/ft_profile.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2109_08219_b200 as dtopk  # noqa: E402
from paper_2109_08219_b200 import data  # noqa: E402

v = data.generate("uniform", 1 << 30, seed=0, device="cuda")
for k in [int(x) for x in (sys.argv[1:] or ["1", "64", "1024", "2048", "4096"])]:
    for _ in range(3):
        dtopk.dr_topk(v, dtopk.PipelineConfig(k=k))
    torch.cuda.synchronize()
    print("k", k, flush=True)
