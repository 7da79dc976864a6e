"""Column-sharded restatement of the CoFEM PCG -- TEST INFRASTRUCTURE ONLY.

Restates, in numpy, the exact exchange pattern the CUDA library implements
for Phi column-sharded across ranks (paper_2105_10439_b200/distributed.py,
csrc/cofem.cu pcg_device): per PCG step an all-reduce of the N x Q partial
Phi_r P_r, an all-reduce of pi, and one of (rho_new, ||R||^2); ||B||^2 and the
initial rho once per solve.  Everything D-indexed stays local.  The
arithmetic follows cg.py:111-152 / kernels.py:27-49 like cofem_oracle.py.
Used by tests/test_distributed.py to check that the sharded decomposition
reproduces the unsharded reference on every rank.

``pcg_solve_time_sharded`` restates the time-sharded convolution path
(csrc/cofem.cu conv_fwd / conv_quantize_v, distributed.time_shards): rank r
holds samples [t0, t1) of P, X, R and of V = Phi P; Phi P takes the left
neighbour's last L-1 samples of P, Phi^T V the right neighbour's first L-1
samples of V (zero at the sequence ends); the PCG scalars are all-reduced.
The convolutions are the reference's (operators.py:182-225) on the local
window, in float64.
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


def _causal_window(taps, window, n_out, adjoint):
    """Valid part of the causal convolution (or its adjoint) over a halo-extended window."""
    L = taps.size
    if not adjoint:  # window = [halo (L-1 rows) | local]; out_i = sum_m h_m w[L-1+i-m]
        full = np.stack([np.convolve(window[:, k], taps)[L - 1:L - 1 + n_out] for k in range(window.shape[1])], 1)
    else:  # window = [local | halo]; out_j = sum_m h_m w[j+m]
        full = np.stack([np.correlate(window[:, k], taps, mode="full")[L - 1:L - 1 + n_out]
                         for k in range(window.shape[1])], 1)
    return full


def pcg_solve_time_sharded(taps, beta, alpha_local, B_local, minv_local, cfg, allreduce, halo):
    """Blocked PCG on this rank's samples of a causal convolution system.

    `halo(rows, direction)` sends `rows` to the neighbour in `direction` (+1:
    right, -1: left) and returns the rows received from the other side
    (zeros at the ends of the chain)."""
    taps = np.asarray(taps, dtype=np.float64)
    L = taps.size
    B = np.asarray(B_local, dtype=np.float64)
    n_loc, ncol = B.shape

    def phi(P):
        left = halo(P[max(n_loc - (L - 1), 0):], +1)  # my tail -> right; the left neighbour's tail -> me
        return _causal_window(taps, np.concatenate([left, P]), n_loc, False)

    def phi_t(V):
        right = halo(V[:L - 1], -1)  # my head -> left; the right neighbour's head -> me
        return _causal_window(taps, np.concatenate([V, right]), n_loc, True)

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
        psi = beta * phi_t(phi(P)) + alpha_local[:, None] * P
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
