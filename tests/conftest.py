"""Shared fixtures.  GPU tests carry @pytest.mark.gpu; the rest run on CPU.

The oracle (oracle/) is imported only here and in tests -- it is the checker.
"""

from __future__ import annotations

import json
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from dtopk_testlib import FIGURE_VECTOR  # noqa: E402

GOLDEN = ROOT / "tests" / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and libdtopk.so")


@pytest.fixture
def figure_vector():
    return FIGURE_VECTOR.copy()


@pytest.fixture
def rng():
    return np.random.default_rng(20240601)


@pytest.fixture(scope="session")
def golden():
    z = np.load(GOLDEN)
    meta = json.loads(bytes(z["__meta__"]).decode())
    return z, meta


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle

    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def assert_multiset_equal(got, expected):
    np.testing.assert_array_equal(np.sort(np.asarray(got).ravel()), np.sort(np.asarray(expected).ravel()))
