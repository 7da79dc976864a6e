"""Rademacher probes and the diagonal estimator rule.

Mirrors /root/reference/pkg/src/sbl/probes.py (draw_rademacher :13-17,
estimate_diagonal_rademacher :28-31).  Inside run_cofem the probes are drawn
on the device (k_pcg64_rademacher reproduces numpy's PCG64
``rng.integers(0, 2)`` stream bit for bit) and the estimator is fused with
the M-step (``k_em_finish``).  The host functions here are the API for
callers that draw or hold probe / solution blocks themselves (explicit
``probe_blocks``, ``e_step``).
"""

from __future__ import annotations

import numpy as np


def draw_rademacher(dim, n_probes, rng):
    """D x K matrix of i.i.d. +-1 entries with equal probability (float64)."""
    if dim < 1 or n_probes < 1:
        raise ValueError("dim and n_probes must be >= 1")
    return rng.integers(0, 2, size=(dim, n_probes)).astype(np.float64) * 2.0 - 1.0


def draw_rademacher_int8(dim, n_probes, rng):
    """Same draw as ``draw_rademacher`` (identical rng consumption) as int8 signs."""
    if dim < 1 or n_probes < 1:
        raise ValueError("dim and n_probes must be >= 1")
    bits = rng.integers(0, 2, size=(dim, n_probes))
    return (bits.astype(np.int8) * 2 - 1).astype(np.int8)


def estimate_diagonal_rademacher(probes, X):
    """s_j = (1/K) sum_k probes_jk X_jk."""
    probes = np.asarray(probes, dtype=np.float64)
    X = np.asarray(X, dtype=np.float64)
    if probes.ndim != 2 or probes.shape != X.shape:
        raise ValueError(f"probes and solutions must share a (D, K) shape, got {probes.shape} vs {X.shape}")
    return np.mean(probes * X, axis=1)
