"""GPU parity: the sm_100a pipeline against the oracle and the reference goldens.

Bar: bit-exact.  Values equal the reference's ``dr_topk`` values; indices equal
the restated tie rule (kernels._extract_exact on V: keys > kth first, then
ties by lowest index; ordered key desc, index asc).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2109_08219_b200 as dtopk
from paper_2109_08219_b200 import data

pytestmark = pytest.mark.gpu


def keys_of(host: np.ndarray, largest: bool, oracle_mod) -> np.ndarray:
    return oracle_mod.to_keys(host, largest)


def check_topk(v_dev: torch.Tensor, k: int, oracle_mod, *, largest=True, **cfgkw):
    """Run dr_topk on device and compare values + indices with the oracle."""
    cfg = dtopk.PipelineConfig(k=k, largest=largest, **cfgkw)
    r = dtopk.dr_topk(v_dev, cfg, exact_stats=True)
    host = v_dev.cpu().numpy()
    keys = keys_of(host, largest, oracle_mod)
    ek, ei = oracle_mod.topk_with_indices(keys, k)
    gi = r.indices.cpu().numpy()
    gv = r.values.cpu().numpy()
    np.testing.assert_array_equal(gi, ei)
    np.testing.assert_array_equal(keys_of(gv, largest, oracle_mod), ek)
    np.testing.assert_array_equal(gv, host[ei])
    # values also equal the reference dr_topk restatement (multiset, order)
    vc = dtopk.validate_config(cfg, host.size)
    ov, ost = oracle_mod.dr_topk(keys, k, vc.alpha, vc.beta, skip_last=False, direct=vc.direct_fallback)
    np.testing.assert_array_equal(keys_of(gv, largest, oracle_mod), ov)
    if not vc.direct_fallback:
        s = r.stats
        assert s.delegate_vector_len == ost.delegate_vector_len
        assert s.fully_qualified_subranges == ost.fully_qualified_subranges
        assert s.partially_qualified_subranges == ost.partially_qualified_subranges
        assert s.concatenated_len == ost.concatenated_len
        assert int(r.stats.device["theta_local"]) == ost.theta
    return r


def test_smoke_entry():
    import __graft_entry__

    __graft_entry__.smoke()


# ---------------------------------------------------------------- delegates
@pytest.mark.parametrize("alpha", [1, 2, 3, 4, 5, 6, 7, 8, 10, 11, 12, 13, 14, 16])
@pytest.mark.parametrize("beta", [1, 2, 3])
def test_delegates_match_oracle(alpha, beta, oracle_mod, cuda):
    if beta >= 1 << alpha:
        pytest.skip("beta must be < 2^alpha")
    for n, dist in [((1 << 20) + 12345, "uniform"), (1 << 19, "few_distinct"), (300_001, "nd_u32")]:
        if (1 << alpha) > n:
            continue
        v = data.generate(dist, n, seed=alpha * 7 + beta, device=cuda)
        d = dtopk.extract_delegates(v, alpha, beta)
        exp = oracle_mod.extract_delegates(v.cpu().numpy(), alpha, beta)
        np.testing.assert_array_equal(d.values.cpu().numpy(), exp)


@pytest.mark.parametrize("beta", [4, 5, 8, 9, 17, 31])
def test_delegates_large_beta(beta, oracle_mod, cuda):
    v = data.generate("uniform", 100_003, seed=beta, device=cuda)
    for alpha in (5, 6, 9):
        if beta >= 1 << alpha:
            continue
        d = dtopk.extract_delegates(v, alpha, beta)
        np.testing.assert_array_equal(d.values.cpu().numpy(), oracle_mod.extract_delegates(v.cpu().numpy(), alpha, beta))


def test_delegate_figure_examples(figure_vector, cuda):
    # pkg/tests/test_delegate.py:16-31 and :55-61
    d = dtopk.extract_delegates(torch.from_numpy(figure_vector).to(cuda), 2, 1)
    assert d.values.cpu().tolist() == [3012, 2313, 3210, 2321]
    d = dtopk.extract_delegates(figure_vector, 2, 2)
    assert d.values[4:6].tolist() == [3210, 3000]
    d = dtopk.extract_delegates(figure_vector, 4, 1)
    assert d.values.tolist() == [3210]
    d = dtopk.extract_delegates(np.array([10, 20, 30, 40, 50], dtype=np.uint32), 2, 2)
    assert d.values.tolist() == [40, 30, 50, 0]
    assert d.tags.tolist() == [0, 0, 1, 1]


# ---------------------------------------------------------------- end to end
@pytest.mark.parametrize("k", [1, 2, 7, 128, 1000, 4096, 1 << 14, 100_000])
@pytest.mark.parametrize("dist", ["uniform", "nd_u32", "few_distinct"])
def test_dr_topk_u32(k, dist, oracle_mod, cuda):
    v = data.generate(dist, (1 << 21) + 3, seed=k % 97, device=cuda)
    check_topk(v, k, oracle_mod)


@pytest.mark.parametrize("dist", ["ascending", "descending", "all_equal"])
@pytest.mark.parametrize("k", [1, 300, 1 << 16])
def test_dr_topk_adversarial(dist, k, oracle_mod, cuda):
    v = data.generate(dist, 1 << 22, seed=1, device=cuda)
    check_topk(v, k, oracle_mod)


@pytest.mark.parametrize("dist,k", [("uniform", 4097), ("uniform", 6000), ("uniform", 8192), ("ascending", 6000),
                                    ("descending", 6000), ("nd_u32", 7000), ("clustered", 6000)])
def test_pass3_one_cta_path(dist, k, oracle_mod, cuda):
    """K2 pass 3's one-CTA path (theta bucket <= 8192 members, select.cuh
    k2_pass3): thread-owned regions, and the warp list for regions above 64
    members ("clustered": every key above 2^31 sits in one block of 20000, so
    the bucket members fill one or two K2 regions)."""
    n = 1 << 22
    if dist == "clustered":
        v = data.generate("uniform", n, seed=5, device=cuda)
        vi = v.view(torch.int32)
        vi &= 0x7FFFFFFF
        vi[n // 2: n // 2 + 20000] |= torch.tensor(-0x80000000, dtype=torch.int32, device=cuda)
    else:
        v = data.generate(dist, n, seed=5, device=cuda)
    check_topk(v, k, oracle_mod)


@pytest.mark.parametrize("k", [20_000, 300_000])
@pytest.mark.parametrize("case", ["uniform", "normal_f32_smallest", "skewed_bucket", "two_values"])
def test_big_answer_sorts(case, k, oracle_mod, cuda):
    """Large answers: bucket sort (uniform, float) and its LSD fallback (a
    bucket above BK_CAP: a block of near-equal keys; two values only)."""
    largest = True
    if case == "uniform":
        v = data.generate("uniform", 1 << 22, seed=k, device=cuda)
    elif case == "normal_f32_smallest":
        v = data.generate("normal_f32", 1 << 22, seed=k, device=cuda)
        largest = False
    elif case == "skewed_bucket":
        v = data.generate("uniform", 1 << 22, seed=k, device=cuda)
        hot = data.generate("uniform", 1 << 22, seed=k + 1, device=cuda).view(torch.int32) & 0xFFF
        v.view(torch.int32)[::5] = (0x7FFFF000 + hot[::5]).to(torch.int32) | torch.iinfo(torch.int32).min
    else:
        v = data.generate("uniform", 1 << 22, seed=k, device=cuda).view(torch.int32) & 1
        v = (v + 7).view(torch.uint32)
    check_topk(v, k, oracle_mod, largest=largest)


@pytest.mark.parametrize("largest", [True, False])
@pytest.mark.parametrize("dist", ["normal_f32", "pareto_f32"])
@pytest.mark.parametrize("beta", [1, 2, 3])
def test_dr_topk_f32(largest, dist, beta, oracle_mod, cuda):
    v = data.generate(dist, 1 << 21, seed=beta, device=cuda)
    check_topk(v, 1024, oracle_mod, largest=largest, beta=beta)


def test_dr_topk_f32_signed_zeros_and_specials(oracle_mod, cuda):
    v = data.generate("normal_f32", 1 << 16, seed=3, device=cuda)
    v[::5] = 0.0
    v[::7] = -0.0
    v[3] = float("inf")
    v[4] = float("-inf")
    for largest in (True, False):
        check_topk(v, 5000, oracle_mod, largest=largest)


@pytest.mark.parametrize("largest", [True, False])
def test_dr_topk_u32_smallest(largest, oracle_mod, cuda):
    v = data.generate("uniform", 1 << 20, seed=5, device=cuda)
    check_topk(v, 777, oracle_mod, largest=largest)


@pytest.mark.parametrize("alpha", [1, 2, 3, 5, 9, 13, 14, 15, 18])
@pytest.mark.parametrize("beta", [1, 2, 3, 8, 12])
def test_dr_topk_manual_alpha_beta(alpha, beta, oracle_mod, cuda):
    v = data.generate("uniform", (1 << 20) + 5, seed=alpha + beta, device=cuda)
    check_topk(v, 333, oracle_mod, alpha=alpha, beta=beta, auto_alpha=False)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 17, 100, 1023, 8191, 8192, 8193, 65537])
def test_dr_topk_small_and_ragged(n, oracle_mod, cuda):
    v = data.generate("uniform", n, seed=n, device=cuda)
    for k in sorted({1, max(1, n // 3), n}):
        check_topk(v, k, oracle_mod)


def test_k_equals_n_sorted(oracle_mod, cuda):
    v = data.generate("uniform", 1024, seed=2, device=cuda)
    r = check_topk(v, 1024, oracle_mod)
    np.testing.assert_array_equal(r.values.cpu().numpy(), np.sort(v.cpu().numpy())[::-1])


def test_direct_fallback(oracle_mod, cuda):
    v = data.generate("uniform", 1024, seed=14, device=cuda)
    r = check_topk(v, 600, oracle_mod, alpha=8, beta=2, auto_alpha=False)
    assert r.stats.delegate_vector_len == 0
    assert set(r.stats.per_stage_nanos) == set(dtopk.STAGES)


def test_numpy_roundtrip_and_ties(oracle_mod, cuda):
    # pkg/tests/test_kernels.py:167-171: [9,5,5,5,9,5], k=3 -> [9,9,5], ties in scan order
    v = np.array([9, 5, 5, 5, 9, 5], dtype=np.uint32)
    r = dtopk.dr_topk(v, dtopk.PipelineConfig(k=3))
    assert isinstance(r.values, np.ndarray)
    assert r.values.tolist() == [9, 9, 5]
    assert r.indices.tolist() == [0, 4, 1]
    assert r.threshold == 5
    # pkg/tests/test_pipeline.py:186-192: duplicated maxima survive filtering
    v = np.zeros(64, dtype=np.uint32)
    v[[3, 17, 33, 49, 5, 21]] = 900
    r = dtopk.dr_topk(v, dtopk.PipelineConfig(k=6, alpha=4, beta=2, auto_alpha=False))
    assert r.values.tolist() == [900] * 6
    assert r.indices.tolist() == [3, 5, 17, 21, 33, 49]


def test_figure_dr_topk(figure_vector, cuda):
    # pkg/tests/test_pipeline.py:60-64
    r = dtopk.dr_topk(figure_vector, dtopk.PipelineConfig(k=2, alpha=2, beta=1, auto_alpha=False))
    assert r.values.tolist() == [3210, 3012]
    assert r.threshold == 3012
    assert r.indices.tolist() == [10, 2]


# ---------------------------------------------------------------- reference goldens
def test_golden_vectors(golden, oracle_mod, cuda):
    z, meta = golden
    for m in meta:
        name, k = m["name"], m["k"]
        v = z[f"{name}__input"]
        if m["kind"] == "u32":
            cfg = dtopk.PipelineConfig(k=k, **m["cfg"])
            r = dtopk.dr_topk(torch.from_numpy(v).to(cuda), cfg, exact_stats=True)
            got = r.values.cpu().numpy()
            np.testing.assert_array_equal(got, z[f"{name}__values_sl1"], err_msg=name)
            np.testing.assert_array_equal(got, z[f"{name}__values_sl0"], err_msg=name)
            assert r.threshold == m["threshold_sl1"], name
            st0 = m["stats_sl0"]
            assert r.stats.delegate_vector_len == st0["delegate_vector_len"], name
            if not m["direct"]:
                assert r.stats.fully_qualified_subranges == st0["fully_qualified_subranges"], name
                assert r.stats.partially_qualified_subranges == st0["partially_qualified_subranges"], name
                assert r.stats.concatenated_len == st0["concatenated_len"], name
                assert int(r.stats.device["theta_local"]) == m["theta_sl0"], name
                d = dtopk.extract_delegates(v, m["alpha"], m["beta"])
                np.testing.assert_array_equal(d.values, z[f"{name}__delegates"], err_msg=name)
        else:
            r = dtopk.dr_topk(v, dtopk.PipelineConfig(k=k, largest=m["largest"]))
            exp = z[f"{name}__values_sl1"]
            np.testing.assert_array_equal(r.values.view(np.uint32), exp.view(np.uint32), err_msg=name)


# ---------------------------------------------------------------- stage mirrors
def test_first_topk_and_concat_mirrors(figure_vector, cuda):
    # pkg/tests/test_pipeline.py:26-58
    d = dtopk.extract_delegates(torch.from_numpy(figure_vector).to(cuda), 2, 1)
    rep = dtopk.first_topk(d, 2, "radix", skip_last=False)
    assert rep.theta == 3012
    assert rep.fully_qualified.cpu().tolist() == [0, 2]
    out = dtopk.concatenate_filtered(torch.from_numpy(figure_vector).to(cuda), rep, 2)
    assert out.cpu().tolist() == [3012, 3210]
    d2 = dtopk.extract_delegates(torch.from_numpy(figure_vector).to(cuda), 2, 2)
    rep = dtopk.first_topk(d2, 3, "radix", skip_last=False)
    assert rep.theta == 3000
    assert rep.fully_qualified.cpu().tolist() == [2]
    assert sorted(rep.partial_values.cpu().tolist()) == [3012]


def test_radix_topk_mirror(oracle_mod, cuda):
    v = data.generate("uniform", 3000, seed=9, device=cuda)
    sel, _, thr = dtopk.radix_topk(v, 99)
    exp = np.sort(v.cpu().numpy())[-99:]
    np.testing.assert_array_equal(np.sort(sel.cpu().numpy()), exp)
    assert thr == int(exp[0])
    assert dtopk.kth_largest(v, 99) == int(exp[0])


@pytest.mark.parametrize("dist", ["uniform", "few_distinct"])
def test_radix_topk_reference_order_and_dtype(dist, cuda):
    """kernels._extract_exact order (kernels.py:83-96): elements above the k-th in
    scan order, then ties in scan order; _extract_at_least (skip_last): every
    element >= the relaxed edge in scan order; values keep the input dtype."""
    v = data.generate(dist, 5000, seed=3, device=cuda)
    h = v.cpu().numpy()
    tags = torch.arange(5000, device=cuda, dtype=torch.int64)
    sel, st, thr = dtopk.radix_topk(v, 300, tags=tags)
    kth = np.sort(h)[-300]
    gt = np.flatnonzero(h > kth)
    idx = np.concatenate([gt, np.flatnonzero(h == kth)[: 300 - gt.size]])
    assert sel.dtype == torch.uint32 and thr == int(kth)
    np.testing.assert_array_equal(sel.cpu().numpy(), h[idx])
    np.testing.assert_array_equal(st.cpu().numpy(), idx)
    sel2, st2, thr2 = dtopk.radix_topk(v, 300, skip_last=True, tags=tags)
    edge = int(kth) & 0xFFFFFF00
    idx2 = np.flatnonzero(h >= edge)
    assert sel2.dtype == torch.uint32 and thr2 == int(h[idx2].min())
    np.testing.assert_array_equal(sel2.cpu().numpy(), h[idx2])
    np.testing.assert_array_equal(st2.cpu().numpy(), idx2)


def test_theta_override_split_path(oracle_mod, cuda):
    """begin/finish with an external theta (the multi-GPU exchange) on one GPU:
    the two halves of a vector, each filtered with max(theta_0, theta_1)."""
    from paper_2109_08219_b200.distributed import DeviceOps

    n, k = 1 << 21, 5000
    v = data.generate("uniform", n, seed=77, device=cuda)
    ops = DeviceOps()
    halves = [v[: n // 2], v[n // 2:]]
    states, thetas = [], []
    for h in halves:
        cfg = dtopk.validate_config(dtopk.PipelineConfig(k=k), h.numel())
        st, th = ops.begin(h, cfg)
        states.append(st)
        thetas.append(th)
    tmax = torch.maximum(thetas[0], thetas[1])
    outs_v, outs_i = [], []
    for r, (st, h) in enumerate(zip(states, halves)):
        vals, idx = ops.finish(st, tmax.clone(), r * (n // 2))
        outs_v.append(vals)
        outs_i.append(idx)
    cat_v = torch.cat(outs_v)
    cat_i = torch.cat(outs_i)
    fv, fi = ops.merge(cat_v, cat_i, k, True)
    ek, ei = oracle_mod.topk_with_indices(v.cpu().numpy(), k)
    np.testing.assert_array_equal(fi.cpu().numpy(), ei)
    np.testing.assert_array_equal(fv.cpu().numpy(), ek)


@pytest.mark.parametrize("dist", ["few_distinct", "all_equal", "nd_u32", "ascending"])
@pytest.mark.parametrize("k", [1, 1000, 1 << 15])
def test_tie_heavy_default_stats_mode(dist, k, oracle_mod, cuda):
    """Default mode (no exact stats): K4T's ordered early stop and K5's
    word skipping must not change values or indices."""
    v = data.generate(dist, (1 << 22) + 77, seed=3, device=cuda)
    r = dtopk.dr_topk(v, dtopk.PipelineConfig(k=k))
    ek, ei = oracle_mod.topk_with_indices(v.cpu().numpy(), k)
    np.testing.assert_array_equal(r.indices.cpu().numpy(), ei)
    np.testing.assert_array_equal(r.values.cpu().numpy(), ek)


@pytest.mark.parametrize("k", [7, 5000, 70000])
def test_graph_plan_replay_matches_eager(k, oracle_mod, cuda):
    from paper_2109_08219_b200 import _native
    from paper_2109_08219_b200.pipeline import DrTopK

    v = data.generate("uniform", 1 << 22, seed=k, device=cuda)
    p = DrTopK(v.numel(), dtopk.PipelineConfig(k=k), _native.DTYPE_U32, torch.uint32, cuda, use_graph=True)
    for _ in range(3):
        p.launch(v)
        torch.cuda.synchronize()
        ek, ei = oracle_mod.topk_with_indices(v.cpu().numpy(), k)
        np.testing.assert_array_equal(p.indices.cpu().numpy(), ei)
        np.testing.assert_array_equal(p.values.cpu().numpy(), ek)
        v.view(torch.int32)[::97] += 1  # new data, same buffer: the plan re-reads it


@pytest.mark.parametrize("k", [5000, 70000])
def test_graph_plan_switches_tie_heavy(k, oracle_mod, cuda):
    """One graph plan replayed over one buffer whose contents switch between
    uniform, tie-heavy and sorted keys: every device-decided path (K2c / K2b on a
    large theta bucket, the pool floor, the graph's conditional tails) follows
    the contents of each launch (api.cu run_finish)."""
    from paper_2109_08219_b200 import _native
    from paper_2109_08219_b200.pipeline import DrTopK

    n = 1 << 22
    buf = torch.empty(n, dtype=torch.uint32, device=cuda)
    p = DrTopK(n, dtopk.PipelineConfig(k=k), _native.DTYPE_U32, torch.uint32, cuda, use_graph=True)
    for dist in ["uniform", "few_distinct", "all_equal", "uniform", "few_distinct", "ascending"]:
        buf.copy_(data.generate(dist, n, seed=3, device=cuda))
        p.launch(buf)
        torch.cuda.synchronize()
        ek, ei = oracle_mod.topk_with_indices(buf.cpu().numpy(), k)
        np.testing.assert_array_equal(p.indices.cpu().numpy(), ei)
        np.testing.assert_array_equal(p.values.cpu().numpy(), ek)


def test_sharded_two_ranks_on_one_gpu(cuda):
    """The multi-rank product path (ShardedTopK and sharded_topk) against the
    oracle with 2 ranks; gloo lets both ranks share this box's single GPU."""
    import os
    import socket
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ, DTOPK_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "tools/dist_check.py"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("dist,largest", [("uniform", True), ("normal_f32", False)])
def test_tuning_sweep_gpu(dist, largest, cuda):
    """Row f3: the sweep harness over an alpha grid and a beta grid, values
    verified against a device sort at every point, reference CSV schema."""
    import io

    from paper_2109_08219_b200 import tuning

    v = data.generate(dist, 1 << 20, seed=11, device=cuda)
    base = dtopk.PipelineConfig(k=128, largest=largest)
    rows = tuning.sweep(v, 128, alphas=[6, 8, 10], base=base, repeats=2)
    assert [r.alpha for r in rows] == [6, 8, 10]
    assert all(r.delegate_len == 2 * ((1 << 20) >> r.alpha) for r in rows)
    assert all(r.total_ns > 0 for r in rows)
    rows_b = tuning.sweep(v, 128, betas=[1, 2, 3], base=base)
    assert [r.beta for r in rows_b] == [1, 2, 3]
    buf = io.StringIO()
    tuning.write_csv(rows + rows_b, buf)
    assert len(buf.getvalue().splitlines()) == 7


@pytest.mark.parametrize("workers,max_resident", [(1, 1 << 26), (3, 1 << 26), (2, 100_000), (4, 65_536)])
def test_run_distributed_streams_partitions(workers, max_resident, oracle_mod, cuda, tmp_path):
    """Rows f1/f2: the partitioned run (reference plan, worker lanes, gather to
    primary); a residency cap below the share streams partitions from the
    DTKV file.  Values and indices against the oracle."""
    n, k = 600_007, 3000
    v = data.gen_uniform(n, 9)
    path = tmp_path / "v.dtkv"
    data.write_vector(path, v)
    rep = dtopk.run_distributed(path, k, workers=workers, max_resident=max_resident)
    ek, ei = oracle_mod.topk_with_indices(v, k)
    np.testing.assert_array_equal(rep.result.values, ek)
    np.testing.assert_array_equal(rep.result.indices, ei)
    plan = dtopk.plan(n, k, workers, max_resident)
    assert rep.reloaded_partitions == sum(1 for p in plan.partitions if not p.resident)
    assert len(rep.messages) == workers and rep.gathered_bytes > 0
    if rep.reloaded_partitions:
        assert sum(m.reload_nanos for m in rep.messages) > 0
    # in-memory source, ties (nd): same answer
    nd = data.gen_normal(200_000, 2)
    rep2 = dtopk.run_distributed(nd, 5000, workers=3, max_resident=30_000)
    ek2, ei2 = oracle_mod.topk_with_indices(nd, 5000)
    np.testing.assert_array_equal(rep2.result.values, ek2)
    np.testing.assert_array_equal(rep2.result.indices, ei2)


def test_cli_gen_run_sweep_dist(cuda, tmp_path, capsys):
    """Row f2: the reference CLI's subcommands and CSV schemas on the GPU path."""
    from paper_2109_08219_b200 import cli, tuning

    f = str(tmp_path / "v.dtkv")
    assert cli.main(["gen", "--dist", "cd", "--n", "2^16", "--k", "100", "--out", f]) == 0
    assert cli.main(["run", f, "--k", "100", "--verify", "--csv", str(tmp_path / "r.csv")]) == 0
    out = capsys.readouterr().out
    assert "verified=true" in out and "ratio_sum=" in out
    assert (tmp_path / "r.csv").read_text().splitlines()[0] == tuning.CSV_HEADER
    assert cli.main(["run", "--dist", "nd", "--n", "2^18", "--k", "2^10", "--verify"]) == 0
    assert cli.main(["sweep", f, "--k", "100", "--param", "alpha", "--grid", "4,6,8",
                     "--csv", str(tmp_path / "s.csv")]) == 0
    assert len((tmp_path / "s.csv").read_text().splitlines()) == 4
    assert cli.main(["dist", f, "--k", "100", "--workers", "3", "--max-resident", "2^13", "--verify",
                     "--csv", str(tmp_path / "d.csv")]) == 0
    lines = (tmp_path / "d.csv").read_text().splitlines()
    assert lines[0] == cli.DIST_CSV_HEADER and len(lines) == 4
    assert cli.main(["run", f, "--k", "0"]) == 2  # InvalidK -> exit 2 (cli.py:270-275)


@pytest.mark.parametrize("seed", range(96))
def test_randomized_configs(seed, oracle_mod, cuda):
    """Property sweep: random n, k, distribution, alpha / beta, largest /
    smallest, u32 / f32 -- values, indices and the reference counters must all
    match the oracle (catches interactions the targeted tests miss)."""
    rng = np.random.default_rng(1000 + seed)
    dist = ["uniform", "few_distinct", "nd_u32", "ascending", "descending", "all_equal", "normal_f32",
            "pareto_f32"][seed % 8]
    n = int(rng.integers(1, 1 << 21)) if seed % 3 else int(rng.integers(1 << 16, 1 << 22))
    k = int(min(n, max(1, rng.choice([1, 7, 100, 1000, 5000, 40000, n // 2]))))
    v = data.generate(dist, n, seed=seed, device=cuda)
    kw = {"largest": bool(seed % 2)}
    if seed % 4 == 1:
        alpha = int(rng.integers(1, max(2, min(18, n.bit_length()))))
        beta = int(rng.integers(1, 6))
        if beta >= (1 << alpha) or beta * -(-n // (1 << alpha)) < k:
            beta = 1
        if beta * -(-n // (1 << alpha)) < k:
            alpha = 1
        if (1 << alpha) > n:
            return
        kw.update(alpha=alpha, beta=beta, auto_alpha=False)
    elif seed % 4 == 2:
        kw.update(beta=int(rng.integers(1, 9)))
    try:
        check_topk(v, k, oracle_mod, **kw)
    except dtopk.InvalidBeta:
        pass


def _key_tensor(v: torch.Tensor, largest: bool) -> torch.Tensor:
    """Device int64 keys of the library's order (larger key = selected first)."""
    b = v.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    if v.dtype == torch.float32:
        b = torch.where(b >> 31 == 1, b ^ 0xFFFFFFFF, b | 0x80000000)
    return b if largest else 0xFFFFFFFF - b


@pytest.mark.parametrize("dist,k,largest", [
    ("uniform", 1, True), ("uniform", 1024, True), ("uniform", 1 << 20, True), ("uniform", 1 << 16, False),
    ("normal_f32", 1024, True), ("ascending", 1 << 16, True), ("nd_u32", 1 << 16, True),
])
def test_full_size_properties(dist, k, largest, cuda):
    """BASELINE sizes (N = 2^30) where the CPU oracle is too slow: size-independent
    properties that pin the answer -- values[i] == v[indices[i]], indices unique,
    (key desc, index asc) order, exactly the keys above the k-th plus the lowest-
    index ties, and the k-th key's rank: #(key > kth) < k <= #(key >= kth)."""
    n = 1 << 30
    v = data.generate(dist, n, seed=5, device=cuda)
    r = dtopk.dr_topk(v, dtopk.PipelineConfig(k=k, largest=largest))
    idx, vals = r.indices, r.values
    assert idx.numel() == k and vals.numel() == k
    assert torch.equal(v.view(torch.int32)[idx], vals.view(torch.int32))
    assert torch.unique(idx).numel() == k
    key = _key_tensor(v, largest)
    kk = key[idx]
    assert bool((kk[:-1] >= kk[1:]).all())
    same = kk[:-1] == kk[1:]
    assert bool((idx[:-1][same] < idx[1:][same]).all())
    kth = int(kk[-1])
    gt = int((key > kth).sum())
    ge = int((key >= kth).sum())
    assert gt < k <= ge
    assert int((kk > kth).sum()) == gt  # every key above the k-th is in the answer
    ties_taken = idx[kk == kth]
    if ties_taken.numel() < ge - gt:  # lowest-index ties first
        all_ties = torch.nonzero(key == kth).flatten()
        assert torch.equal(torch.sort(ties_taken).values, all_ties[: ties_taken.numel()])
    del key, v
    torch.cuda.empty_cache()


def test_config5_single_gpu_2pow33_properties(cuda):
    """BASELINE config 5 size on one GPU (N = 2^33, 32 GiB): answer properties,
    with the rank counts of the k-th key taken chunk by chunk."""
    n, k = 1 << 33, 1024
    v = data.generate("uniform", n, seed=9, device=cuda)
    r = dtopk.dr_topk(v, dtopk.PipelineConfig(k=k))
    idx = r.indices
    vi = v.view(torch.int32)
    assert torch.equal(vi[idx], r.values.view(torch.int32))
    assert torch.unique(idx).numel() == k
    kk = vi[idx].to(torch.int64) & 0xFFFFFFFF
    assert bool((kk[:-1] >= kk[1:]).all())
    same = kk[:-1] == kk[1:]
    assert bool((idx[:-1][same] < idx[1:][same]).all())
    kth = int(kk[-1])
    gt = ge = 0
    ties = []
    for c in range(0, n, 1 << 30):
        ch = vi[c:c + (1 << 30)].to(torch.int64) & 0xFFFFFFFF
        gt += int((ch > kth).sum())
        ge += int((ch >= kth).sum())
        ties.append(torch.nonzero(ch == kth).flatten() + c)
        del ch
    assert gt < k <= ge
    assert int((kk > kth).sum()) == gt  # every key above the k-th is in the answer
    # lowest-index ties first: the taken kth ties are the first ones in index order
    taken = torch.sort(idx[kk == kth]).values
    all_ties = torch.cat(ties)
    assert torch.equal(taken, all_ties[: taken.numel()])
    del v, vi
    torch.cuda.empty_cache()
