"""GPU parity of the stage-level API (the reference's operators) against the
oracle / numpy restatements of pipeline.py:87-159 and delegate.py:93-127.

* ``first_topk``: theta (kernels.radix_topk, exact and skip_last-relaxed) and
  the qualification report (selected / partial delegates with tags, fully
  qualified subranges) through ``dtopk_kth_largest`` / ``dtopk_min_at_least``
  / ``dtopk_qualify``;
* ``concatenate_filtered`` through ``dtopk_concat``;
* beta > 32 delegates (``k1_bigbeta``) and a full dr_topk with beta = 40.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2109_08219_b200 as dtopk
from paper_2109_08219_b200 import data

pytestmark = pytest.mark.gpu


def _np_qualify(D: np.ndarray, beta: int, theta: int):
    """pipeline.py:104-116 restated."""
    tags = np.repeat(np.arange(D.size // beta), beta)
    in_t = D >= theta
    per = np.bincount(tags[in_t], minlength=D.size // beta)
    full = per == beta
    partial = in_t & ~full[tags]
    return D[in_t], tags[in_t], np.flatnonzero(full), D[partial], tags[partial]


@pytest.mark.parametrize("alpha,beta,k,skip_last", [(6, 2, 5000, False), (6, 2, 5000, True), (8, 1, 300, True),
                                                    (10, 3, 2000, False), (11, 2, 64, True), (5, 4, 40000, False)])
@pytest.mark.parametrize("dist", ["uniform", "few_distinct"])
def test_first_topk_matches_reference(alpha, beta, k, skip_last, dist, oracle_mod, cuda):
    v = data.generate(dist, (1 << 22) + 77, seed=alpha + beta, device=cuda)
    d = dtopk.extract_delegates(v, alpha, beta)
    D = d.values.cpu().numpy().astype(np.uint32) if isinstance(d.values, torch.Tensor) else np.asarray(d.values)
    if k > D.size:
        pytest.skip("k beyond |D|")
    theta = oracle_mod.radix_threshold(D, k, skip_last)
    rep = dtopk.first_topk(d, k, "radix", skip_last=skip_last)
    assert rep.theta == theta
    sv, st, fq, pv, pt = _np_qualify(D, beta, theta)
    np.testing.assert_array_equal(rep.selected_values.cpu().numpy(), sv)
    np.testing.assert_array_equal(rep.selected_tags.cpu().numpy(), st)
    np.testing.assert_array_equal(rep.fully_qualified.cpu().numpy(), fq)
    np.testing.assert_array_equal(rep.partial_values.cpu().numpy(), pv)
    np.testing.assert_array_equal(rep.partial_tags.cpu().numpy(), pt)
    out = dtopk.concatenate_filtered(v, rep, alpha)
    host = v.cpu().numpy()
    W = 1 << alpha
    exp = np.concatenate([host[s * W:(s + 1) * W][host[s * W:(s + 1) * W] >= theta] for s in fq]) if fq.size else \
        np.empty(0, np.uint32)
    np.testing.assert_array_equal(out.cpu().numpy(), exp)


def test_concat_float32_keys(oracle_mod, cuda):
    """concatenate_filtered on float32 input compares in key space (the
    order-preserving map) and returns float32 values."""
    v = data.generate("normal_f32", 1 << 20, seed=4, device=cuda)
    d = dtopk.extract_delegates(v, 7, 2)
    rep = dtopk.first_topk(d, 500, "radix", skip_last=False)
    out = dtopk.concatenate_filtered(v, rep, 7).cpu().numpy()
    host = v.cpu().numpy()
    keys = oracle_mod.to_keys(host, True)
    W = 1 << 7
    fq = rep.fully_qualified.cpu().numpy()
    exp = np.concatenate([host[s * W:(s + 1) * W][keys[s * W:(s + 1) * W] >= rep.theta] for s in fq])
    assert out.dtype == np.float32
    np.testing.assert_array_equal(out.view(np.uint32), exp.view(np.uint32))


@pytest.mark.parametrize("alpha,beta", [(6, 40), (8, 100), (10, 33), (13, 500)])
def test_delegates_beta_above_32(alpha, beta, oracle_mod, cuda):
    v = data.generate("uniform", (1 << 20) + 13, seed=beta, device=cuda)
    d = dtopk.extract_delegates(v, alpha, beta)
    exp = oracle_mod.extract_delegates(v.cpu().numpy(), alpha, beta)
    got = d.values.cpu().numpy() if isinstance(d.values, torch.Tensor) else np.asarray(d.values)
    np.testing.assert_array_equal(got.astype(np.uint32), exp)


@pytest.mark.parametrize("dist", ["uniform", "few_distinct", "all_equal"])
def test_dr_topk_beta_40(dist, oracle_mod, cuda):
    from test_gpu_parity import check_topk

    v = data.generate(dist, (1 << 21) + 5, seed=40, device=cuda)
    check_topk(v, 3000, oracle_mod, alpha=9, auto_alpha=False, beta=40)


# ---------------------------------------------------------------- streamed host input (row f1)
@pytest.mark.parametrize("kind,n,k,largest,dtype", [
    ("numpy", (1 << 25) + 4099, 1000, True, "u32"),      # pageable: pinned staging, 3 ranges, ragged tail
    ("numpy", 1 << 25, 1, True, "u32"),                  # alpha > 11: k1_merge after the last range
    ("pinned", (1 << 24) + 2048, 70000, False, "u32"),   # pinned: direct DMA per range
    ("torch_cpu", (1 << 24) + 5, 3000, True, "f32"),
])
def test_streamed_host_input(kind, n, k, largest, dtype, oracle_mod, cuda):
    from paper_2109_08219_b200 import _device

    g = data.generate("normal_f32" if dtype == "f32" else "uniform", n, seed=n % 97, device=cuda)
    host = g.cpu()
    if kind == "pinned":
        host = host.pin_memory()
    v = host.numpy() if kind == "numpy" else host
    assert n >= _device.STREAM_MIN
    r = dtopk.dr_topk(v, dtopk.PipelineConfig(k=k, largest=largest))
    keys = oracle_mod.to_keys(host.numpy(), largest)
    ek, ei = oracle_mod.topk_with_indices(keys, k)
    gi = np.asarray(r.indices.numpy() if isinstance(r.indices, torch.Tensor) else r.indices)
    gv = np.asarray(r.values.numpy() if isinstance(r.values, torch.Tensor) else r.values)
    np.testing.assert_array_equal(gi, ei)
    np.testing.assert_array_equal(oracle_mod.to_keys(gv, largest), ek)
    # counters equal the resident-input call's
    r2 = dtopk.dr_topk(g, dtopk.PipelineConfig(k=k, largest=largest))
    for f in ("delegate_vector_len", "fully_qualified_subranges", "partially_qualified_subranges"):
        assert getattr(r.stats, f) == getattr(r2.stats, f), f
