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


def ref_spread(solve, rhs, seeds=8):
    """The reference's own iteration-count spread under rounding-level input
    changes (checker side): `solve(b)` runs the reference solver
    and returns its iteration count; it is called on `rhs` and on `seeds`
    copies of it multiplied element-wise by (1 + 2^-52 u), u ~ U(-1, 1).
    BiCGSTAB counts are rounding-chaotic (the reference's own
    -O2 and FMA builds take 211 and 75 iterations at 50^2), so a GPU count is
    judged against this spread, not against one sample.  Returns (min, max)."""
    counts = [solve(rhs)]
    for sd in range(seeds):
        u = np.random.default_rng(sd).uniform(-1.0, 1.0, rhs.size)
        counts.append(solve(rhs * (1.0 + np.ldexp(u, -52))))
    return min(counts), max(counts)


def within_spread(it, lo, hi, slack=0.05):
    """[0.95 min, 1.05 max] of the reference's spread."""
    return (1.0 - slack) * lo <= it <= (1.0 + slack) * hi
