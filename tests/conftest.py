import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libmpbjac.so")
    config.addinivalue_line("markers", "slow: full-size configuration runs")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


def golden_cases(g):
    """Matrix cases of the fixture (every key group that carries a matrix)."""
    return sorted({k.split("/")[0] for k in g if k.endswith("/row_ptr")})


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    from paper_2407_15973_b200 import _lib
    _lib.load()
    return torch.device("cuda", 0)


def dense_to_csr(a, dtype=np.float64):
    """SparseMatrix from a dense array, dropping exact zeros (the reference
    test helper, pkg/tests/conftest.py:20-25)."""
    from paper_2407_15973_b200 import SparseMatrix
    a = np.asarray(a, dtype=dtype)
    rows, cols = np.nonzero(a)
    return SparseMatrix.from_coo(a.shape[0], a.shape[1], rows, cols, a[rows, cols], dtype=dtype)


def random_spd_csr(n, density, rng, dtype=np.float64):
    """Random symmetric diagonally dominant CSR (pkg/tests/conftest.py:28-34)."""
    a = rng.uniform(-1.0, 1.0, size=(n, n))
    a[rng.uniform(size=(n, n)) > density] = 0.0
    a = a + a.T
    np.fill_diagonal(a, np.abs(a).sum(axis=1) + 1.0)
    return dense_to_csr(a, dtype=dtype)
