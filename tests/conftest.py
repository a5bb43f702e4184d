import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the native kernels")


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def assert_rel(got, ref, rtol, floor=1e-30, what=""):
    """Per entry |got-ref| <= rtol*|ref| (+ a denormal floor), zeros exact."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    err = np.abs(got - ref)
    bad = err > rtol * np.abs(ref) + floor
    assert not bad.any(), (
        f"{what}: {int(bad.sum())} entries outside rtol={rtol}; worst rel "
        f"{float((err / np.maximum(np.abs(ref), 1e-300)).max()):.3e}")
    zero = ref == 0.0
    assert np.all(got[zero] == 0.0), f"{what}: {int((got[zero] != 0).sum())} nonzeros where ref == 0"


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch
