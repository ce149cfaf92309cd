import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref/libsdcore_ref.so) -- checker only."""
    from oracle.refpy import RefLib
    return RefLib()


@pytest.fixture(scope="session")
def port():
    """The plain-C restatement (oracle/_ref/liboracle_port.so) -- checker only."""
    from oracle.refpy import PortLib
    return PortLib()


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    return load


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_2108_13229_b200 import sdc
    return sdc.default_context()


def to_sdc(a):
    """oracle Csr -> product SparseMatrix."""
    from paper_2108_13229_b200.sdc import SparseMatrix
    return SparseMatrix(a.n_rows, a.n_cols, a.rowptr, a.col, a.val)


def golden_csr(g, prefix, n_rows, n_cols=None):
    from oracle.refpy import Csr
    return Csr(n_rows, n_rows if n_cols is None else n_cols, g[f"{prefix}_rowptr"], g[f"{prefix}_col"],
               g[f"{prefix}_val"])


def rel_l2(x, y):
    return float(np.linalg.norm(np.asarray(x) - np.asarray(y)) / max(np.linalg.norm(y), 1e-300))


def bitwise_equal(x, y):
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    # -0.0 and +0.0 are the same value; everything else must match bit for bit
    return x.shape == y.shape and bool(np.all((x.view(np.uint64) == y.view(np.uint64)) | ((x == 0) & (y == 0))))
