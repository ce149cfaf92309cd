"""IQN-ILS interface quasi-Newton update of the partitioned driver, restated
from /root/reference/proj/core/src/coupling.cpp:12-101 (IqnIlsHistory,
iqn_ils_update).  Host-side O(interface x history) work, as in the reference
(it stays host).  Loops keep the reference's operation order
(sequential dot / axpy, MGS with one reorthogonalisation pass, column
filtering, back substitution), so the update is bitwise the reference's for
the same inputs.
"""
from __future__ import annotations

from typing import List, Optional

import numpy as np


def _dot(a: np.ndarray, b: np.ndarray) -> float:
    s = 0.0
    for x, y in zip(a.tolist(), b.tolist()):
        s += x * y
    return s


def _norm2(a: np.ndarray) -> float:
    return float(np.sqrt(_dot(a, a)))


class IqnIlsHistory:
    """coupling.hpp:38-76: difference columns, newest first, at most
    min(capacity, interface dimension) of them."""

    def __init__(self, capacity: int = 50, filter_tolerance: float = 1e-13):
        self.capacity = capacity
        self.filter_tolerance = filter_tolerance
        self.prev_residual: Optional[np.ndarray] = None
        self.prev_v_tilde: Optional[np.ndarray] = None
        self.d_residual: List[np.ndarray] = []
        self.d_v_tilde: List[np.ndarray] = []

    def has_previous(self) -> bool:
        return self.prev_residual is not None

    def record(self, residual, v_tilde):
        self.prev_residual = np.array(residual, dtype=np.float64)
        self.prev_v_tilde = np.array(v_tilde, dtype=np.float64)

    def push(self, residual, v_tilde):
        if not self.has_previous():
            raise ValueError("iqn-ils: no prior iterate stored")
        residual = np.asarray(residual, dtype=np.float64)
        v_tilde = np.asarray(v_tilde, dtype=np.float64)
        self.d_residual.insert(0, residual - self.prev_residual)
        self.d_v_tilde.insert(0, v_tilde - self.prev_v_tilde)
        limit = min(self.capacity, residual.size)
        del self.d_residual[limit:]
        del self.d_v_tilde[limit:]
        self.record(residual, v_tilde)


def iqn_ils_update(history: IqnIlsHistory, v_k, residual_k, v_tilde_k1) -> np.ndarray:
    """coupling.cpp:45-101: v_{k+1} = v_k + R_k + What alpha with alpha the
    least-squares solution of min ||Vhat alpha + R_k|| (QR by MGS2, filtered)."""
    if not history.has_previous():
        raise ValueError("iqn-ils: no prior iterate stored")
    history.push(residual_k, v_tilde_k1)
    residual_k = np.asarray(residual_k, dtype=np.float64)
    q: List[np.ndarray] = []
    r_cols: List[List[float]] = []
    kept: List[int] = []
    for c, col in enumerate(history.d_residual):
        w = col.copy()
        norm0 = _norm2(w)
        rc = [0.0] * (len(kept) + 1)
        for _ in range(2):
            for k in range(len(q)):
                proj = _dot(w, q[k])
                rc[k] += proj
                w = w + (-proj) * q[k]
        wn = _norm2(w)
        if norm0 == 0.0 or wn <= history.filter_tolerance * norm0:
            continue
        rc[-1] = wn
        w = w * (1.0 / wn)
        q.append(w)
        r_cols.append(rc)
        kept.append(c)
    nk = len(kept)
    g = [-_dot(residual_k, q[k]) for k in range(nk)]
    alpha = [0.0] * nk
    for i in range(nk - 1, -1, -1):
        s = g[i]
        for j in range(i + 1, nk):
            s -= r_cols[j][i] * alpha[j]
        alpha[i] = s / r_cols[i][i]
    v_next = np.asarray(v_k, dtype=np.float64) + residual_k
    for k in range(nk):
        v_next = v_next + alpha[k] * history.d_v_tilde[kept[k]]
    return v_next
