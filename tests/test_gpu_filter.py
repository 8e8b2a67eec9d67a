"""GPU parity of the filtered delegate pass (K0 sample -> K1 records -> K2 over
records, csrc/delegate.cuh / select.cuh) and of its fallback.

For alpha 6..8 and beta <= 2, K1 stores only the subranges whose max delegate
reaches a floor sampled from 1/128 of the K1 chunks; K2 checks that the floor
lies at or below theta's first-digit bucket and otherwise re-runs the full K1 +
K2.  Either way the answer must equal the oracle's bit for bit (values,
indices, the reference counters of pipeline.py:87-159).  The fallback is forced
with inputs whose sampled chunks hold the largest keys, so the sample
overestimates theta.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2109_08219_b200 as dtopk
from paper_2109_08219_b200 import _native, data
from paper_2109_08219_b200.pipeline import DrTopK

from test_gpu_parity import check_topk

pytestmark = pytest.mark.gpu

K0_GROUP = 512
K0_REGIONS = 64
CHUNK = 2048


def sampled_chunks(n: int) -> np.ndarray:
    """K1 chunks K0 samples (k0_sample: 64 runs of L = max(1, nch / 32768) consecutive
    full chunks, run r at r * (nch / 64) + a hashed offset)."""
    nch = n // CHUNK
    slot, L = nch // K0_REGIONS, max(1, nch // (K0_REGIONS * K0_GROUP))
    r = np.arange(K0_REGIONS, dtype=np.uint64)
    h = ((r.astype(np.uint32) * np.uint32(0x9E3779B1)) >> np.uint32(16)).astype(np.uint64) % np.uint64(slot - L + 1)
    start = r * np.uint64(slot) + h
    return (start[:, None] + np.arange(L, dtype=np.uint64)[None, :]).ravel().astype(np.int64)


def adversarial_for_sample(n: int, alpha: int, cuda, dtype=torch.uint32):
    """Uniform keys below 2^31, except the sampled chunks, lifted above 2^31."""
    v = data.generate("uniform", n, seed=3, device=cuda)
    vi = v.view(torch.int32)
    vi &= 0x7FFFFFFF
    cs = torch.from_numpy(sampled_chunks(n)).to(cuda)
    rows = vi[: (n // CHUNK) * CHUNK].view(-1, CHUNK)
    rows[cs] |= torch.tensor(-0x80000000, dtype=torch.int32, device=cuda)
    return v


def header(r):
    return r.stats.device


@pytest.mark.parametrize("alpha,k", [(6, 4096), (7, 3000), (8, 1000), (6, 8192)])
@pytest.mark.parametrize("beta", [1, 2])
def test_filtered_pass_matches_oracle(alpha, k, beta, oracle_mod, cuda):
    n = (1 << 24) + 4099  # ragged tail chunk and tail subrange
    v = data.generate("uniform", n, seed=alpha * 7 + beta, device=cuda)
    r = check_topk(v, k, oracle_mod, alpha=alpha, auto_alpha=False, beta=beta)
    assert header(r)["filtered"] == 1 and header(r)["filter_fallback"] == 0


@pytest.mark.parametrize("largest", [True, False])
def test_filtered_pass_f32(largest, oracle_mod, cuda):
    """float32 at alpha 7 (the first digit is log-scale from the top of the key
    range, so N(0,1) keys may share one bucket and keep the filter off: parity
    either way)."""
    v = data.generate("normal_f32", 1 << 24, seed=5, device=cuda)
    check_topk(v, 30000, oracle_mod, largest=largest, alpha=7, auto_alpha=False)


@pytest.mark.parametrize("alpha,k", [(6, 20000), (8, 4000)])
def test_filter_fallback_eager(alpha, k, oracle_mod, cuda):
    v = adversarial_for_sample(1 << 24, alpha, cuda)
    r = check_topk(v, k, oracle_mod, alpha=alpha, auto_alpha=False)
    assert header(r)["filtered"] == 1 and header(r)["filter_fallback"] == 1


def test_filter_fallback_graph_plan(oracle_mod, cuda):
    """The fallback as a conditional node of the plan's CUDA graph; the same plan
    then replays on data where the sample is representative (no fallback)."""
    n, alpha, k = 1 << 24, 6, 20000
    v = adversarial_for_sample(n, alpha, cuda)
    cfg = dtopk.PipelineConfig(k=k, alpha=alpha, auto_alpha=False)
    p = DrTopK(n, cfg, _native.DTYPE_U32, torch.uint32, cuda, use_graph=True)
    for adversarial in (True, False, True):
        v.copy_(adversarial_for_sample(n, alpha, cuda) if adversarial else data.generate("uniform", n, seed=9,
                                                                                         device=cuda))
        p.launch(v)
        torch.cuda.synchronize()
        keys = v.cpu().numpy()
        ek, ei = oracle_mod.topk_with_indices(keys, k)
        np.testing.assert_array_equal(p.indices.cpu().numpy(), ei)
        np.testing.assert_array_equal(p.values.cpu().numpy(), ek)
        assert int(p.header().filter_fallback) == (1 if adversarial else 0)


def test_filter_off_on_ties(oracle_mod, cuda):
    """Tie-heavy input: the sampled bucket holds most of the sample, the filter
    stays off and the full pass runs."""
    v = data.generate("few_distinct", 1 << 24, seed=1, device=cuda)
    r = check_topk(v, 1 << 15, oracle_mod, alpha=6, auto_alpha=False)
    assert header(r)["filtered"] == 0


def test_sharded_begin_uses_filter(oracle_mod, cuda):
    """dtopk_select_begin / finish (the multi-GPU split) with the filtered pass."""
    n, k = 1 << 24, 1 << 15
    v = data.generate("uniform", n, seed=12, device=cuda)
    cfg = dtopk.validate_config(dtopk.PipelineConfig(k=k, alpha=6, auto_alpha=False), n)
    p = DrTopK(n, cfg, _native.DTYPE_U32, torch.uint32, cuda, timed=False)
    s = torch.cuda.current_stream()
    lib = p.lib
    _native.check(lib.dtopk_select_begin(v.data_ptr(), n, _native.DTYPE_U32, k, 1, cfg.alpha, cfg.beta, 0,
                                         p.ws.data_ptr(), p.ws_bytes, s.cuda_stream, None), "begin")
    _native.check(lib.dtopk_select_finish(v.data_ptr(), n, _native.DTYPE_U32, k, 1, cfg.alpha, cfg.beta, 0, None,
                                          p.values.data_ptr(), p.indices.data_ptr(), 0, p.ws.data_ptr(), p.ws_bytes,
                                          s.cuda_stream, None), "finish")
    torch.cuda.synchronize()
    ek, ei = oracle_mod.topk_with_indices(v.cpu().numpy(), k)
    np.testing.assert_array_equal(p.indices.cpu().numpy(), ei)
    assert int(p.header().filtered) == 1


# ---------------------------------------------------------------- pool floor (K4h)
@pytest.mark.parametrize("case,k,largest", [
    ("ascending", 1 << 14, True),        # 4 M keys above theta, floor keeps ~k
    ("ascending_dups", 1 << 14, True),   # every key 4 times: ties straddle the floor's bin
    ("descending", 1 << 14, False),      # smallest of a descending vector: the same shape mirrored
    ("ascending_f32", 8192, True),
])
def test_pool_floor(case, k, largest, oracle_mod, cuda):
    """Calls that re-read >= 2M keys above theta take the pool floor: values,
    indices and the reference counters (|C| included) stay exact, and the pool
    shrinks to about k."""
    n = 1 << 24
    if case == "ascending_f32":
        v = torch.arange(n, device=cuda, dtype=torch.float32) - n / 2
    elif case == "ascending_dups":
        v = (torch.arange(n, device=cuda, dtype=torch.int64) // 4).to(torch.int32).view(torch.uint32)
    else:
        v = data.generate(case, n, seed=0, device=cuda)
    alpha = 10 if case == "ascending_f32" else 9
    r = check_topk(v, k, oracle_mod, largest=largest, alpha=alpha, auto_alpha=False)
    assert int(r.stats.device["pool_gt"]) < 4 * k  # the floor cut the pool (millions of keys above theta)
