"""Reference-named helpers (shardkrp/reference.py:15-68), kept for API parity.

``dense_mttkrp_oracle`` keeps its name and contract (validation, messages,
float64 (I_mode, R) result) but is computed on the GPU like every other
MTTKRP in this package -- the independent CPU restatement used as the parity
checker lives outside the product, in ``oracle/`` at the repository root.
"""

from __future__ import annotations

import numpy as np

from .engine import mttkrp


def khatri_rao(m1, m2) -> np.ndarray:
    """Column-wise Kronecker product; rows sweep m2's rows fastest."""
    m1 = np.asarray(m1)
    m2 = np.asarray(m2)
    if m1.ndim != 2 or m2.ndim != 2:
        raise ValueError("khatri_rao expects 2-D matrices")
    if m1.shape[1] != m2.shape[1]:
        raise ValueError(f"column count mismatch: {m1.shape[1]} vs {m2.shape[1]}")
    return (m1[:, None, :] * m2[None, :, :]).reshape(m1.shape[0] * m2.shape[0], m1.shape[1])


def dense_mttkrp_oracle(tensor, factors, mode: int) -> np.ndarray:
    """dense_mttkrp_oracle's contract, computed by the GPU engine."""
    return mttkrp(tensor, factors, mode)
