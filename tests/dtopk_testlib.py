"""Shared test constants (uniquely named: a foreign `tests` package exists on this image)."""

from __future__ import annotations

import pathlib

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent

# The reference's 16-element worked example (pkg/tests/conftest.py:10-18):
# four subranges of four; subrange 2's top two are {3210, 3000}.
FIGURE_VECTOR = np.array(
    [101, 2001, 3012, 1323, 2313, 878, 1500, 450, 3000, 1002, 3210, 2500, 2321, 700, 1900, 1100],
    dtype=np.uint32,
)
