"""Shared fixtures.  `gpu` marks tests that need a B200 (run with -m gpu)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_golden(name: str):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated yet")
    return np.load(path, allow_pickle=False)


@pytest.fixture(scope="session")
def ref_small():
    return load_golden("ref_small.npz")


def small_cases(g):
    for i in range(int(g["n_cases"])):
        k = f"c{i}_"
        yield i, {name[len(k):]: g[name] for name in g.files if name.startswith(k)}


@pytest.fixture(scope="session")
def gp():
    """The product package with its native library (GPU tests only)."""
    import paper_2007_16076_b200 as pkg
    from paper_2007_16076_b200 import _lib

    _lib.load_library()
    return pkg


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.lib()
    return O
