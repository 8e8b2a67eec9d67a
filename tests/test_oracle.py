"""CPU: the oracle (oracle/) pinned against the reference's own outputs.

Golden vectors come from the unmodified reference package (see
tests/golden/make_golden.py); the reference's own known-answer tests are
restated at the bottom (pkg/tests/test_delegate.py, test_pipeline.py,
test_kernels.py).
"""

from __future__ import annotations

import numpy as np
import pytest

from dtopk_testlib import FIGURE_VECTOR


def test_golden_dr_topk_values_and_stats(golden, oracle_mod):
    z, meta = golden
    checked = 0
    for m in meta:
        if m["kind"] != "u32":
            continue
        v = z[f"{m['name']}__input"]
        for tag, sl in (("sl1", True), ("sl0", False)):
            vals, st = oracle_mod.dr_topk(v, m["k"], m["alpha"], m["beta"], skip_last=sl, direct=m["direct"])
            np.testing.assert_array_equal(vals, z[f"{m['name']}__values_{tag}"], err_msg=m["name"])
            exp = m[f"stats_{tag}"]
            got = {f: getattr(st, f) for f in exp}
            assert got == exp, (m["name"], tag, got, exp)
            assert int(vals[-1]) == m[f"threshold_{tag}"]
            checked += 1
    assert checked >= 40


def test_golden_delegates_and_theta(golden, oracle_mod):
    z, meta = golden
    for m in meta:
        if m["kind"] != "u32" or m["direct"]:
            continue
        v = z[f"{m['name']}__input"]
        d = oracle_mod.extract_delegates(v, m["alpha"], m["beta"])
        np.testing.assert_array_equal(d, z[f"{m['name']}__delegates"], err_msg=m["name"])
        np.testing.assert_array_equal(oracle_mod.np_extract_delegates(v, m["alpha"], m["beta"]), d)
        for tag, sl in (("sl1", True), ("sl0", False)):
            assert oracle_mod.radix_threshold(d, m["k"], sl) == m[f"theta_{tag}"], m["name"]
            assert oracle_mod.np_radix_threshold(d, m["k"], sl) == m[f"theta_{tag}"], m["name"]


def test_golden_float_and_smallest_via_key_map(golden, oracle_mod):
    z, meta = golden
    n = 0
    for m in meta:
        if m["kind"] != "f32":
            continue
        v = z[f"{m['name']}__input"]
        keys = oracle_mod.to_keys(v, m["largest"])
        cfg_alpha = oracle_mod.auto_alpha(v.size, m["k"])
        vals, _ = oracle_mod.dr_topk(keys, m["k"], cfg_alpha, min(2, (1 << cfg_alpha) - 1))
        got = oracle_mod.from_keys(vals, np.float32, m["largest"])
        np.testing.assert_array_equal(got.view(np.uint32), z[f"{m['name']}__values_sl1"].view(np.uint32))
        n += 1
    assert n == 6


def test_key_map_is_order_preserving(oracle_mod):
    x = np.array([-np.inf, -3.5, -1e-30, -0.0, 0.0, 1e-30, 2.0, np.inf], dtype=np.float32)
    k = oracle_mod.to_keys(x, True)
    assert np.all(np.diff(k.astype(np.int64)) > 0)
    assert np.array_equal(oracle_mod.from_keys(k, np.float32, True).view(np.uint32), x.view(np.uint32))
    ks = oracle_mod.to_keys(x, False)
    assert np.all(np.diff(ks.astype(np.int64)) < 0)


@pytest.mark.parametrize("dist", ["uniform", "few", "equal", "asc"])
def test_index_oracle_matches_lexsort(dist, oracle_mod, rng):
    n = 50_000
    if dist == "uniform":
        v = rng.integers(0, 2**32, n, dtype=np.uint32)
    elif dist == "few":
        v = rng.integers(0, 16, n, dtype=np.uint32)
    elif dist == "equal":
        v = np.full(n, 7, dtype=np.uint32)
    else:
        v = np.arange(n, dtype=np.uint32)
    for k in (1, 17, 1000, n):
        ok, oi = oracle_mod.topk_with_indices(v, k)
        ek, ei = oracle_mod.np_topk_with_indices(v, k)
        np.testing.assert_array_equal(oi, ei)
        np.testing.assert_array_equal(ok, ek)


def test_oracle_random_instances_vs_numpy(oracle_mod, rng):
    """Random restatement cross-check (the reference's soundness style,
    pkg/tests/test_acceptance.py:63-87): values equal the sorted oracle."""
    for _ in range(200):
        n = int(rng.integers(2, 3000))
        v = rng.integers(0, int(rng.choice([5, 1000, 2**32])), n, dtype=np.uint32)
        alpha = int(rng.integers(1, n.bit_length()))
        beta = int(rng.integers(1, 4))
        if beta >= 1 << alpha:
            continue
        s = -(-n // (1 << alpha))
        k = int(rng.integers(1, min(beta * s, n) + 1))
        vals, _ = oracle_mod.dr_topk(v, k, alpha, beta, skip_last=bool(rng.integers(0, 2)))
        np.testing.assert_array_equal(vals, np.sort(v)[::-1][:k])


def test_partitioned_oracle_equals_single(oracle_mod):
    v = oracle_mod.generate_uniform(1 << 18, seed=3)
    single, _ = oracle_mod.dr_topk(v, 128, oracle_mod.auto_alpha(v.size, 128), 2)
    for w in (1, 2, 4, 8):
        np.testing.assert_array_equal(oracle_mod.dr_topk_partitioned(v, 128, w), single)


# ---- the reference's known-answer tests, restated on the oracle
def test_reference_figure_examples(oracle_mod):
    v = FIGURE_VECTOR
    assert oracle_mod.extract_delegates(v, 2, 1).tolist() == [3012, 2313, 3210, 2321]  # test_delegate.py:16-20
    assert oracle_mod.extract_delegates(v, 2, 2)[4:6].tolist() == [3210, 3000]  # :22-26
    assert oracle_mod.extract_delegates(v, 4, 1).tolist() == [3210]  # :28-31
    tail = np.array([10, 20, 30, 40, 50], dtype=np.uint32)
    assert oracle_mod.extract_delegates(tail, 2, 2).tolist() == [40, 30, 50, 0]  # :55-61
    d = oracle_mod.extract_delegates(v, 2, 1)
    assert oracle_mod.radix_threshold(d, 2, False) == 3012  # test_pipeline.py:26-33
    vals, st = oracle_mod.dr_topk(v, 2, 2, 1, skip_last=False)
    assert vals.tolist() == [3210, 3012] and st.fully_qualified_subranges == 2  # :60-64
    d2 = oracle_mod.extract_delegates(v, 2, 2)
    assert oracle_mod.radix_threshold(d2, 3, False) == 3000  # :51-58
    ties = np.array([9, 5, 5, 5, 9, 5], dtype=np.uint32)
    ok, oi = oracle_mod.topk_with_indices(ties, 3)  # test_kernels.py:167-171
    assert ok.tolist() == [9, 9, 5] and oi.tolist() == [0, 4, 1]


def test_generator_host_twin(oracle_mod):
    from paper_2109_08219_b200 import data

    a = data.generate_host("uniform", 5000, seed=9, offset=17)
    b = oracle_mod.generate_uniform(5000, seed=9, offset=17)
    np.testing.assert_array_equal(a, b)
    assert np.array_equal(data.generate_host("ascending", 10), np.arange(10, dtype=np.uint32))
    f = data.generate_host("few_distinct", 4096, seed=1)
    assert f.max() < 16 and len(np.unique(f)) == 16
