"""Column-sharded restatement of the CoFEM PCG -- TEST INFRASTRUCTURE ONLY.

Restates, in numpy, the exact exchange pattern the CUDA library implements
for Phi column-sharded across ranks (paper_2105_10439_b200/distributed.py,
csrc/cofem.cu pcg_device): per PCG step an all-reduce of the N x Q partial
Phi_r P_r, an all-reduce of pi, and one of (rho_new, ||R||^2); ||B||^2 and the
initial rho once per solve.  Everything D-indexed stays local.  The
arithmetic follows cg.py:111-152 / kernels.py:27-49 like cofem_oracle.py.
Used by tests/test_distributed.py to check that the sharded decomposition
reproduces the unsharded reference on every rank.
"""

from __future__ import annotations

import numpy as np

from .cofem_oracle import CgConfig, CgReport, DivergenceError, _safe_ratio


def pcg_solve_sharded(phi_local, beta, alpha_local, B_local, minv_local, cfg, allreduce):
    """Blocked PCG on this rank's columns; `allreduce(np.ndarray) -> np.ndarray` sums over ranks."""
    B = np.asarray(B_local, dtype=np.float64)
    ncol = B.shape[1]
    minv = np.asarray(minv_local, dtype=np.float64)[:, None]
    X = np.zeros_like(B)
    bn2 = allreduce((B * B).sum(axis=0))
    bnorm = np.sqrt(bn2.sum())
    if bnorm == 0.0:
        return CgReport(X, 0, 0.0, True)
    if 1.0 <= cfg.tolerance:
        return CgReport(X, 0, 1.0, True)
    R = B.copy()
    P = np.zeros_like(B)
    rho = np.ones(ncol)

    def direction():
        nonlocal P, rho
        W = R * minv
        rho_new = allreduce(np.einsum("jq,jq->q", R, W))
        eta = _safe_ratio(rho_new, rho)
        P = P * eta + (R if cfg.printed_recursion else W)
        rho = rho_new

    direction()
    delta, steps = 1.0, 0
    for u in range(1, cfg.max_steps + 1):
        V = allreduce(phi_local @ P)                       # the N x Q exchange
        psi = beta * (phi_local.T @ V) + alpha_local[:, None] * P
        pi = allreduce(np.einsum("jq,jq->q", P, psi))
        gamma = _safe_ratio(rho, pi)
        X += P * gamma
        R -= psi * gamma
        rn2 = allreduce(np.einsum("jq,jq->q", R, R))
        steps = u
        delta = float(np.sqrt(rn2.sum()) / bnorm)
        if not np.isfinite(delta):
            raise DivergenceError(u)
        if delta <= cfg.tolerance:
            break
        if u < cfg.max_steps:
            direction()
    return CgReport(X, steps, delta, delta <= cfg.tolerance)
