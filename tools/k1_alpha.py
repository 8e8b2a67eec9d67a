"""K1 alone (dtopk_extract_delegates) on 2^30 uniform keys for each alpha.

    DTOPK_LIB=... python tools/k1_alpha.py [alphas...]

CUDA events around 20 back-to-back launches after 3 warm-ups; prints ms and
the read roofline 4N/t per alpha.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2109_08219_b200 import _native, data  # noqa: E402

lib = _native.load()
n = 1 << 30
v = data.generate("uniform", n, seed=0, device="cuda")
s = torch.cuda.current_stream()
for alpha in [int(x) for x in (sys.argv[1:] or ["6", "7", "8", "9", "10", "11"])]:
    beta = 2
    S = -(-n >> alpha)
    wsb = lib.dtopk_workspace_bytes(n, 1, alpha, beta, 0)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    out = torch.empty(S * beta, dtype=torch.int32, device="cuda")

    def run():
        _native.check(lib.dtopk_extract_delegates(v.data_ptr(), n, _native.DTYPE_U32, 1, alpha, beta, out.data_ptr(),
                                                  ws.data_ptr(), wsb, s.cuda_stream), "extract")
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"alpha {alpha}: {ms:.4f} ms  {4 * n / ms / 1e6:.0f} GB/s", flush=True)
    del ws, out
