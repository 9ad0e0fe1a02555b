"""Shared fixtures. `gpu`-marked tests call the CUDA path through the C ABI and
compare it with the oracle (oracle/_ref = the reference itself, or the plain-C
port oracle/_build); everything else runs on the CPU."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs on the B200 box)")


@pytest.fixture(scope="session")
def ilug():
    import paper_2111_09512_b200 as m
    return m


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle
    if not os.path.exists(oracle.REF_SO):
        pytest.skip("oracle/_ref not built (reference sources unavailable)")
    return oracle.Ref()


@pytest.fixture(scope="session")
def port():
    from oracle import oracle
    if not os.path.exists(oracle.PORT_SO):
        oracle.build(ref=False)
    return oracle.Port()


@pytest.fixture(scope="session")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device (no CPU fallback exists)"
    torch.cuda.set_device(0)
    return torch


def rel_err(a, b):
    """Norm-wise relative error (tests/oracles.hpp:83-90)."""
    a, b = np.asarray(a), np.asarray(b)
    den = np.linalg.norm(b)
    num = np.linalg.norm(a - b)
    return num / den if den > 0 else num


def bitwise(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))
