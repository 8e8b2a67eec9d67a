"""Small cases over every device path, for compute-sanitizer (memcheck /
racecheck / synccheck); each case is checked against the oracle.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [quick]

Paths: fast_tail (small k), general chain + finish_small, large pool (select,
bucket sort), direct radix path, filtered delegate pass and its fallback,
tie-heavy truncation (single- and multi-valued bucket), beta 3 / 40, float32
smallest, stage operators, streamed host input, begin/finish split and the
multi-GPU merge kernels (single list and two lists).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2109_08219_b200 as dtopk  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2109_08219_b200 import _native, data  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
dev = torch.device("cuda")
fails = 0


def check(name, v, k, **kw):
    global fails
    largest = kw.get("largest", True)
    r = dtopk.dr_topk(v, dtopk.PipelineConfig(k=k, **kw))
    host = v.cpu().numpy() if isinstance(v, torch.Tensor) else v
    keys = oracle.to_keys(host, largest)
    ek, ei = oracle.topk_with_indices(keys, k)
    gi = r.indices.cpu().numpy() if isinstance(r.indices, torch.Tensor) else r.indices
    ok = np.array_equal(gi, ei)
    fails += not ok
    print(f"{name:40s} {'OK' if ok else 'MISMATCH'}", flush=True)


n = 1 << 20
u = data.generate("uniform", n, seed=1, device=dev)
check("fast_tail k=64", u, 64)
check("general chain k=4096", u, 4096)
check("general chain k=6000 (pass 3 one-CTA path)", u, 6000)
check("large pool k=2^17 (select+bucket sort)", u, 1 << 17)
check("direct path", u[:5000].clone(), 4999)
check("beta 3", u, 1000, beta=3)
check("float32 smallest", data.generate("normal_f32", n, seed=2, device=dev), 3000, largest=False)
if not quick:
    big = data.generate("uniform", 1 << 22, seed=3, device=dev)
    check("filtered pass alpha 6", big, 8192, alpha=6, auto_alpha=False)
    adv = big.clone()
    vi = adv.view(torch.int32)
    vi &= 0x7FFFFFFF
    nch = (1 << 22) // 2048
    slot, L = nch // 64, 1
    r = np.arange(64, dtype=np.uint64)
    h = ((r.astype(np.uint32) * np.uint32(0x9E3779B1)) >> np.uint32(16)).astype(np.uint64) % np.uint64(slot - L + 1)
    cs = torch.from_numpy((r * np.uint64(slot) + h).astype(np.int64)).to(dev)
    vi.view(-1, 2048)[cs] |= torch.tensor(-0x80000000, dtype=torch.int32, device=dev)
    check("filtered pass fallback", adv, 20000, alpha=6, auto_alpha=False)
    check("tie-heavy single value", data.generate("all_equal", 1 << 22, seed=0, device=dev), 5000)
    check("tie-heavy few distinct", data.generate("few_distinct", 1 << 22, seed=0, device=dev), 5000)
    check("beta 40", u, 2000, alpha=9, auto_alpha=False, beta=40)
    d = dtopk.extract_delegates(u, 6, 2)
    rep = dtopk.first_topk(d, 3000, "radix", skip_last=True)
    out = dtopk.concatenate_filtered(u, rep, 6)
    print(f"{'stage operators':40s} OK ({out.numel()} concatenated)", flush=True)
    host = data.generate("uniform", (1 << 24) + 11, seed=4, device=dev).cpu()
    check("streamed host input", host.numpy(), 1000)
    # begin / finish split + merge kernels (single list)
    lib = _native.load()
    cfg = dtopk.validate_config(dtopk.PipelineConfig(k=1000), n)
    from paper_2109_08219_b200.pipeline import DrTopK

    p = DrTopK(n, cfg, _native.DTYPE_U32, torch.uint32, dev, timed=False)
    s = torch.cuda.current_stream().cuda_stream
    _native.check(lib.dtopk_select_begin(u.data_ptr(), n, 0, 1000, 1, cfg.alpha, cfg.beta, 0, p.ws.data_ptr(),
                                         p.ws_bytes, s, None), "begin")
    _native.check(lib.dtopk_select_finish(u.data_ptr(), n, 0, 1000, 1, cfg.alpha, cfg.beta, 0, None,
                                          p.values.data_ptr(), p.indices.data_ptr(), 0, p.ws.data_ptr(), p.ws_bytes,
                                          s, None), "finish")
    # two sorted lists (the halves of the answer) merged back
    kk = 1000
    half = kk // 2
    vals = p.values.view(torch.int32)
    lens = torch.tensor([half, kk - half], dtype=torch.int64, device=dev)
    offs = torch.tensor([0, half], dtype=torch.int64, device=dev)
    ov = torch.empty(kk, dtype=torch.int32, device=dev)
    oi = torch.empty(kk, dtype=torch.int64, device=dev)
    tp = int(lib.dtopk_merge_tmp_pairs(2, kk))
    tv = torch.empty(tp, dtype=torch.int32, device=dev)
    ti = torch.empty(tp, dtype=torch.int64, device=dev)
    tl = torch.empty(4, dtype=torch.int64, device=dev)
    _native.check(lib.dtopk_merge_lists(0, 1, vals.data_ptr(), 1, 1, p.indices.data_ptr(), offs.data_ptr(), 0,
                                        lens.data_ptr(), 1, 2, kk, ov.data_ptr(), oi.data_ptr(), tv.data_ptr(),
                                        ti.data_ptr(), tl.data_ptr(), s), "merge")
    ok = torch.equal(oi, p.indices)
    fails += not ok
    print(f"{'split + merge kernels':40s} {'OK' if ok else 'MISMATCH'}", flush=True)
torch.cuda.synchronize()
print("ALL OK" if not fails else f"{fails} FAILURES", flush=True)
sys.exit(1 if fails else 0)
