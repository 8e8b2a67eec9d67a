"""CPU: host-side drop-in logic and the C-ABI boundary (no GPU compute).

Config semantics restate the reference's pkg/tests/test_core.py and
test_tuning.py anchors; the boundary tests check that libdtopk.so loads and
exports every symbol include/dtopk.h declares.
"""

from __future__ import annotations

import ctypes
import re

import numpy as np
import pytest

import paper_2109_08219_b200 as dtopk
from paper_2109_08219_b200 import _native
from paper_2109_08219_b200.core import (
    EmptyInput,
    InvalidBeta,
    InvalidK,
    PipelineConfig,
    WorkloadStats,
    delegate_vector_len,
    effective_beta,
    validate_config,
)
from dtopk_testlib import ROOT


class TestValidateConfig:
    def test_auto_alpha_anchors(self):
        # test_core.py:22-30, test_tuning.py:67-91
        assert validate_config(PipelineConfig(k=2**24), 2**30).alpha == 4
        assert validate_config(PipelineConfig(k=2**19), 2**30).alpha == 7
        assert dtopk.auto_alpha(2**30, 2**24) == 4
        assert dtopk.auto_alpha(2**30, 2**19) == 7
        assert dtopk.auto_alpha(2**24, 2**10) == 8
        # the bench sweep
        for k, a in [(1, 16), (2**7, 13), (2**10, 11), (2**13, 10), (2**16, 8), (2**18, 7), (2**20, 6)]:
            assert validate_config(PipelineConfig(k=k), 2**30).alpha == a

    def test_alpha_ignored_unless_auto_alpha_false(self):
        # core.py:165 quirk kept: PipelineConfig(k=5, alpha=3) re-tunes
        assert validate_config(PipelineConfig(k=5, alpha=3), 1000).alpha == 5
        assert validate_config(PipelineConfig(k=5, alpha=3, auto_alpha=False), 1000).alpha == 3

    def test_fallbacks(self):
        assert validate_config(PipelineConfig(k=1, alpha=0, auto_alpha=False), 1).direct_fallback
        assert validate_config(PipelineConfig(k=2**10), 2**10).direct_fallback
        assert validate_config(PipelineConfig(k=100, alpha=6, beta=2, auto_alpha=False), 1024).direct_fallback

    def test_clamps(self):
        assert validate_config(PipelineConfig(k=4, alpha=2, beta=9, auto_alpha=False), 64).beta == 3
        assert validate_config(PipelineConfig(k=2, alpha=30, auto_alpha=False), 64).alpha == 6
        assert effective_beta(2, 0) == 1 and effective_beta(2, 1) == 1 and effective_beta(9, 3) == 7

    def test_idempotent(self):
        for k, n, alpha, auto in [(7, 500, None, True), (3, 64, 4, False), (64, 64, 1, False)]:
            once = validate_config(PipelineConfig(k=k, alpha=alpha, auto_alpha=auto), n)
            assert validate_config(once, n) == once

    def test_errors(self):
        with pytest.raises(InvalidK):
            validate_config(PipelineConfig(k=0), 10)
        with pytest.raises(InvalidK):
            validate_config(PipelineConfig(k=11), 10)
        with pytest.raises(EmptyInput):
            validate_config(PipelineConfig(k=1), 0)
        with pytest.raises(InvalidBeta):
            validate_config(PipelineConfig(k=1, beta=0), 10)
        with pytest.raises(InvalidK):
            validate_config(PipelineConfig(k=100, backend="bitonic"), 1024)
        with pytest.raises(ValueError):
            validate_config(PipelineConfig(k=1, backend="quick"), 10)
        validate_config(PipelineConfig(k=128, backend="bitonic"), 1024)

    def test_matches_reference_formula_against_oracle(self, oracle_mod, rng):
        for _ in range(300):
            n = int(rng.integers(1, 2**31))
            k = int(rng.integers(1, n + 1))
            beta = int(rng.integers(1, 5))
            assert dtopk.auto_alpha(n, k, beta=beta) == oracle_mod.auto_alpha(n, k, 3.0, beta)


def test_delegate_len_formula(rng):
    for _ in range(50):
        n = int(rng.integers(1, 10_000))
        alpha = int(rng.integers(0, n.bit_length()))
        beta = int(rng.integers(1, 5))
        assert delegate_vector_len(n, alpha, beta) == beta * -(-n // (1 << alpha))


def test_stats_thread_safe():
    import threading

    stats = WorkloadStats()

    def bump():
        for _ in range(10_000):
            stats.add_read(1)
            stats.add_written(2)
            stats.add_stage_nanos("FirstK", 3)

    ts = [threading.Thread(target=bump) for _ in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert stats.elements_read == 40_000 and stats.elements_written == 80_000
    assert stats.total_nanos() == 120_000


def test_public_names_match_reference_surface():
    # the drop-in exports the reference's hot-path names (pkg/src/dtopk/__init__.py)
    for name in ["PipelineConfig", "TopKResult", "WorkloadStats", "DtopkError", "InvalidK", "EmptyInput",
                 "InvalidBeta", "validate_config", "dr_topk", "first_topk", "concatenate_filtered",
                 "extract_delegates", "extract_delegates_blocked", "DelegateVector", "radix_topk",
                 "auto_alpha", "plan", "WorkerFailed", "BACKENDS", "ELEMENT_DTYPE", "KeyedEntry",
                 "QualificationReport", "PartitionPlan"]:
        assert hasattr(dtopk, name), name


# ---------------------------------------------------------------- C-ABI boundary
def _header_symbols():
    text = (ROOT / "include" / "dtopk.h").read_text()
    return sorted(set(re.findall(r"\b(dtopk_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    syms = _header_symbols()
    assert "dtopk_select" in syms and len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) <= set(_native.EXPORTS), set(syms) - set(_native.EXPORTS)


def test_library_host_only_entry_points():
    lib = _native.load(require_cuda=False)
    assert lib.dtopk_version().startswith(b"dtopk-b200")
    assert lib.dtopk_result_offset() == 0
    assert ctypes.sizeof(_native.DtopkResult) == 112
    # workspace sizing is host arithmetic
    ws1 = lib.dtopk_workspace_bytes(1 << 30, 1024, 11, 2, 0)
    ws2 = lib.dtopk_workspace_bytes(1 << 30, 1 << 20, 6, 2, 0)
    assert 0 < ws1 < ws2 < 8 * 2**30
    assert lib.dtopk_workspace_bytes(1 << 20, 600, 0, 1, 1) > 0


def test_status_codes_raise_reference_exceptions():
    with pytest.raises(EmptyInput):
        _native.check(_native.EMPTY_INPUT, "x")
    with pytest.raises(InvalidK):
        _native.check(_native.INVALID_K, "x")
    with pytest.raises(InvalidBeta):
        _native.check(_native.INVALID_BETA, "x")
    with pytest.raises(ValueError):
        _native.check(_native.INVALID_ARG, "x")
    with pytest.raises(RuntimeError):
        _native.check(_native.CUDA_ERROR, "x")
    _native.check(_native.OK, "x")


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(_native.NativeUnavailable):
        dtopk.dr_topk(np.arange(100, dtype=np.uint32), PipelineConfig(k=5))


def test_plan_arithmetic():
    # pkg/tests/test_distributed.py:17-52
    p = dtopk.plan(2**26, 128, workers=4, max_resident=2**26)
    assert len(p.partitions) == 4 and p.partition_len == 2**24
    assert all(x.resident for x in p.partitions)
    p = dtopk.plan(2**28, 128, workers=2, max_resident=2**26)
    assert p.assignments == {0: [0, 2], 1: [1, 3]}
    assert [x.resident for x in p.partitions] == [True, True, False, False]
    with pytest.raises(InvalidK):
        dtopk.plan(2**20, 2**19, workers=8, max_resident=2**26)
    assert dtopk.shard_bounds(10, 3, 2) == (8, 2)
    assert sum(dtopk.shard_bounds(1_000_003, 7, r)[1] for r in range(7)) == 1_000_003


def test_tuning_cost_model_and_csv_schema():
    """Row f3 mirror: the reference cost model (tuning.py:61-71), its convex
    argmin near Eq. 11, and the sweep CSV schema (tuning.py:33-36, 189-201)."""
    import io
    import math

    from paper_2109_08219_b200 import tuning

    n, k = 1 << 20, 128
    c = tuning.model_cost(8, k, n)
    inv, size = 2.0 ** -8, 2.0 ** 8
    assert c.t_delegate == (1 + inv) * n + 31 * n * inv
    assert c.t_firstk == 5 * n * inv + 2 * k
    assert c.t_concat == k + 2 * k * size
    assert c.t_secondk == 4 * k * size
    assert c.total == c.t_delegate + c.t_firstk + c.t_concat + c.t_secondk
    totals = {a: tuning.model_cost(a, k, n).total for a in range(1, 20)}
    best = min(totals, key=totals.get)
    assert abs(best - 0.5 * (math.log2(n) - math.log2(k) + 2.62)) <= 1.0
    with pytest.raises(ValueError):
        tuning.CostModelParams(c_global=0)
    row = tuning.SweepRow(8, 2, 128, n, 1, 2, 3, 4, 10, 8192, 2)
    buf = io.StringIO()
    tuning.write_csv([row], buf)
    assert buf.getvalue() == tuning.CSV_HEADER + "\n8,2,128,1048576,1,2,3,4,10,8192,2\n"
    assert tuning.CSV_HEADER.split(",")[0] == "alpha" and len(tuning.CSV_HEADER.split(",")) == 11
    # b200_const inverts Eq. 11 for exact optima
    assert abs(tuning.b200_const({(1 << 30, 1024): 11}) - (2 * 11.5 - 30 + 10)) < 1e-9


def test_reference_generators_and_vector_file(tmp_path):
    """Rows a11 / f1: the reference's ud / nd / cd generators and the DTKV file
    format, against vectors and file bytes the unmodified reference produced
    (tests/golden/make_gen_golden.py)."""
    import os

    from paper_2109_08219_b200 import data

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "gen_golden.npz"))
    np.testing.assert_array_equal(data.generate("ud", 4096, 7), g["ud_4096_7"])
    np.testing.assert_array_equal(data.generate("nd", 4096, 7), g["nd_4096_7"])
    np.testing.assert_array_equal(data.generate("cd", 16384, 3, k=100), g["cd_16384_3"])
    p = tmp_path / "v.dtkv"
    data.write_vector(p, g["ud_4096_7"][:333])
    assert p.read_bytes() == g["dtkv_bytes"].tobytes()
    assert data.read_header(p) == 333
    np.testing.assert_array_equal(data.read_vector(p, offset=5, count=100), g["ud_4096_7"][5:105])
    buf = np.empty(50, dtype=np.uint32)
    data.read_vector(p, offset=300, count=33, out=buf)
    np.testing.assert_array_equal(buf[:33], g["ud_4096_7"][300:333])
    bad = tmp_path / "bad.dtkv"
    bad.write_bytes(b"XXXX" + p.read_bytes()[4:])
    with pytest.raises(data.BadMagic):
        data.read_header(bad)
    bad.write_bytes(p.read_bytes()[:-4])
    with pytest.raises(data.TruncatedFile):
        data.read_header(bad)
    with pytest.raises(data.InfeasibleN):
        data.gen_customized(100, 1, 0)
    with pytest.raises(ValueError):
        data.read_vector(p, offset=300, count=100)


def test_cli_parser_and_counts():
    """Row f2 host side: count notation and the reference's subcommand set."""
    from paper_2109_08219_b200 import cli

    assert cli.parse_count("2^24") == 1 << 24 and cli.parse_count(" 77 ") == 77
    assert cli.parse_grid("2^4,5, 6") == [16, 5, 6]
    p = cli.build_parser()
    a = p.parse_args(["sweep", "--dist", "ud", "--n", "2^20", "--k", "128", "--param", "beta", "--grid", "1,2,3"])
    assert a.command == "sweep" and a.param == "beta" and a.const == 3.0 and a.backend == "radix"
    a = p.parse_args(["dist", "x.dtkv", "--k", "10", "--workers", "4"])
    assert a.max_resident == str(1 << 26)
    with pytest.raises(SystemExit):
        p.parse_args(["run", "--k", "1", "--backend", "heap"])


def test_host_view_coercion():
    """Host inputs of dr_topk's streamed path: the reference's
    np.asarray(v, dtype=uint32) coercion, float32 kept, CUDA tensors excluded."""
    import numpy as np
    import torch

    from paper_2109_08219_b200 import _device, _native
    from paper_2109_08219_b200.core import EmptyInput

    hv = _device.host_view([3, 1, 2])
    assert hv.code == _native.DTYPE_U32 and hv.kind == "numpy" and hv.host.tolist() == [3, 1, 2]
    hv = _device.host_view(np.array([-1, 5], dtype=np.int64))
    assert hv.host.view(torch.int32).tolist() == [-1, 5]  # wrapped to uint32 bits like np.asarray(.., uint32)
    hv = _device.host_view(np.arange(4, dtype=np.float32))
    assert hv.code == _native.DTYPE_F32 and hv.host.dtype == torch.float32
    hv = _device.host_view(torch.arange(5, dtype=torch.int32))
    assert hv.kind == "torch_cpu" and hv.out_dtype == torch.int32 and hv.n == 5
    with pytest.raises(EmptyInput):
        _device.host_view(np.array([], dtype=np.uint32))
    assert _device.STREAM_RANGE % 2048 == 0  # ranges are whole K1 chunks
