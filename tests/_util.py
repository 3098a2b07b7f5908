"""Shared test helpers (importable as `_util`; tests/ is on sys.path under pytest)."""

import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")

#: parity bar: max|y - y_ref| <= 1e-12 * max|y_ref|
PARITY_TOL = 1e-12


def normwise(a, b):
    """max|a-b| / max|b| — the parity metric."""
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))
