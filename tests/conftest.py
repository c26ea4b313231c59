"""Shared fixtures and the `gpu` marker.

CPU tier (`-m "not gpu"`): oracle vs golden vectors from the reference, host
logic, C-ABI symbol table, multi-process (gloo) sharding logic.
GPU tier (`-m gpu`): parity of the sm_100a path against the oracle / goldens.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz") as f:
        return {k: f[k] for k in f.files}


@pytest.fixture(scope="session")
def golden_projector():
    return load_golden("projector")


@pytest.fixture(scope="session")
def golden_warps():
    return load_golden("warps")


@pytest.fixture(scope="session")
def golden_sampling():
    return load_golden("sampling")


@pytest.fixture(scope="session")
def golden_tiny():
    return load_golden("solver_tiny")


@pytest.fixture(scope="session")
def golden_c1():
    return load_golden("solver_c1")


@pytest.fixture()
def rng():
    return np.random.default_rng(1234)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
