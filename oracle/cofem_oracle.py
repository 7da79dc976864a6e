"""Numpy restatement of the reference CoFEM path -- TEST INFRASTRUCTURE ONLY.

Not product code: see ``oracle/__init__.py``.  Every function cites the
reference file:line it restates (paths relative to
/root/reference/pkg/src/sbl/).  Arithmetic is float64 by default, exactly
like the reference; ``dtype=np.float32`` runs the same recursions in single
precision, which the parity tests use to size the fp32 tolerance band.

Parity: pinned against golden vectors produced by the real reference
(tests/golden/make_golden.py -> tests/golden/*.npz).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from scipy.fft import dct, idct, irfft, next_fast_len, rfft
from scipy.special import erfcx

# ----------------------------------------------------------------------------
# seeded streams and probes


def substream(seed, *key):
    """problem.py:10-16 -- child generator keyed by SeedSequence([seed, *key])."""
    return np.random.default_rng(np.random.SeedSequence([int(seed)] + [int(k) for k in key]))


def draw_rademacher(dim, n_probes, rng):
    """probes.py:13-17 -- D x K matrix of +-1 from rng.integers(0, 2)."""
    if dim < 1 or n_probes < 1:
        raise ValueError("dim and n_probes must be >= 1")
    bits = rng.integers(0, 2, size=(dim, n_probes))
    return bits.astype(np.float64) * 2.0 - 1.0


def estimate_diagonal_rademacher(probes, X):
    """probes.py:28-31 -- s_j = (1/K) sum_k p_jk x_jk."""
    probes = np.asarray(probes, dtype=np.float64)
    X = np.asarray(X, dtype=np.float64)
    if probes.shape != X.shape or probes.ndim != 2:
        raise ValueError("probes and solutions must share a (D, K) shape")
    return (probes * X).sum(axis=1) / probes.shape[1]


# ----------------------------------------------------------------------------
# operators (operators.py): each is a small dict of closures over float64 data


@dataclass
class Op:
    n_rows: int
    n_cols: int
    apply: object          # (D, Q) -> (N, Q)
    adjoint: object        # (N, Q) -> (D, Q)
    col_sq_norms: object   # () -> (D,)
    materialize: object    # () -> (N, D)
    kind: str = "dense"


def dense_op(matrix):
    """operators.py:104-129 -- explicit dense Phi; apply = Phi @ V."""
    m = np.array(matrix, dtype=np.float64)
    return Op(
        m.shape[0],
        m.shape[1],
        lambda V: m @ V,
        lambda U: m.T @ U,
        lambda: np.einsum("ij,ij->j", m, m),
        lambda: m.copy(),
        "dense",
    )


def dct_op(dim, mask):
    """operators.py:132-179 -- Phi = rows `mask` of the inverse orthonormal DCT-II."""
    mask = np.sort(np.asarray(mask, dtype=np.int64))

    def fwd(V):
        return idct(V, axis=0, norm="ortho")[mask, :]

    def adj(U):
        full = np.zeros((dim, U.shape[1]))
        full[mask, :] = U
        return dct(full, axis=0, norm="ortho")

    def norms():
        # column j of Phi: c_j cos(pi (2 m_i + 1) j / (2 D)), operators.py:165-179
        pts = (2.0 * mask + 1.0) * (np.pi / (2.0 * dim))
        out = np.empty(dim)
        for lo in range(0, dim, 512):
            hi = min(lo + 512, dim)
            c = np.cos(np.outer(np.arange(lo, hi), pts))
            out[lo:hi] = (c * c).sum(axis=1)
        out *= 2.0 / dim
        out[0] *= 0.5
        return out

    return Op(mask.size, dim, fwd, adj, norms,
              lambda: idct(np.eye(dim), axis=0, norm="ortho")[mask, :], "dct")


def dct2_op(n, mask):
    """BASELINE config 4 (the 2-D analogue of operators.py:132-179): rows `mask`
    of the orthonormal 2-D DCT-II of n x n images flattened row-major."""
    from scipy.fft import dctn, idctn

    mask = np.sort(np.asarray(mask, dtype=np.int64))
    D = n * n

    def fwd(V):
        Y = dctn(V.reshape(n, n, V.shape[1]), axes=(0, 1), norm="ortho")
        return Y.reshape(D, V.shape[1])[mask]

    def adj(U):
        full = np.zeros((D, U.shape[1]))
        full[mask] = U
        return idctn(full.reshape(n, n, U.shape[1]), axes=(0, 1), norm="ortho").reshape(D, U.shape[1])

    def norms():
        k = np.arange(n)[:, None]
        i = np.arange(n)[None, :]
        c = np.cos(np.pi * (2 * i + 1) * k / (2.0 * n)) * np.where(k == 0, np.sqrt(1.0 / n), np.sqrt(2.0 / n))
        g = np.zeros(D)
        g[mask] = 1.0
        return ((c * c).T @ g.reshape(n, n) @ (c * c)).ravel()

    return Op(mask.size, D, fwd, adj, norms, lambda: fwd(np.eye(D)), "dct2")


def conv_op(dim, taps):
    """operators.py:182-225 -- causal lower-triangular Toeplitz convolution.

    The reference's filter is taps[m] = (1 - rho)^m for m < D; a shorter
    `taps` vector is a truncated filter (BASELINE config 3).  FFT path with
    zero padding >= D + L - 1, as the reference's rfft/irfft path.
    """
    taps = np.asarray(taps, dtype=np.float64)
    L = taps.size
    pad = next_fast_len(dim + L - 1)
    spec = rfft(taps, pad)

    def fwd(V):
        return irfft(rfft(V, pad, axis=0) * spec[:, None], pad, axis=0)[:dim]

    def adj(U):
        return irfft(rfft(U, pad, axis=0) * np.conj(spec)[:, None], pad, axis=0)[:dim]

    def norms():
        # column j holds taps[0 : min(L, D - j)]
        c = np.concatenate([[0.0], np.cumsum(taps * taps)])
        lengths = np.minimum(L, dim - np.arange(dim))
        return c[lengths]

    def mat():
        m = np.zeros((dim, dim))
        for j in range(dim):
            n = min(L, dim - j)
            m[j:j + n, j] = taps[:n]
        return m

    return Op(dim, dim, fwd, adj, norms, mat, "conv")


def system_apply(op, beta, alpha, V):
    """operators.py:267-272 -- A V = beta Phi^T (Phi V) + diag(alpha) V."""
    return beta * op.adjoint(op.apply(V)) + alpha[:, None] * V


# ----------------------------------------------------------------------------
# blocked PCG (cg.py + kernels.py)


class DivergenceError(RuntimeError):
    """cg.py:17-26 -- non-finite residual, carries the step index."""

    def __init__(self, step, context=""):
        msg = f"non-finite residual at CG step {step}"
        if context:
            msg = f"{msg} ({context})"
        super().__init__(msg)
        self.step = step


@dataclass(frozen=True)
class CgConfig:
    """cg.py:48-67."""

    max_steps: int = 400
    tolerance: float = 1e-4
    theta_policy: object = "all-ones"
    printed_recursion: bool = False


@dataclass(frozen=True)
class CgReport:
    """cg.py:70-76."""

    solution: np.ndarray
    steps_taken: int
    final_relative_residual: float
    converged: bool
    breakdown_columns: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))


def make_preconditioner(policy, op, beta, alpha):
    """cg.py:79-108 -- diagonal m = beta theta + alpha (or ones for 'none')."""
    alpha = np.asarray(alpha, dtype=np.float64)
    if not np.all(alpha > 0):
        raise ValueError("alpha entries must all be positive")
    if isinstance(policy, str):
        if policy == "none":
            return np.ones(op.n_cols)
        if policy == "all-ones":
            theta = np.ones(op.n_cols)
        elif policy == "jacobi":
            theta = op.col_sq_norms()
        else:
            raise ValueError(f"unknown theta policy {policy!r}")
    else:
        theta = np.asarray(policy, dtype=np.float64)
        if theta.shape != (op.n_cols,) or not np.all(theta > 0):
            raise ValueError("custom theta must be a positive length-D vector")
    return beta * theta + alpha


def _safe_ratio(num, den):
    """num/den where den != 0, else 0 (kernels.py:33 and :47)."""
    out = np.zeros_like(num)
    np.divide(num, den, out=out, where=den != 0.0)
    return out


def pcg_solve(apply_fn, B, minv, cfg, dtype=np.float64):
    """cg.py:111-152 (+ kernels.py:29-52): lockstep blocked PCG.

    minv is (D,) or (D, Q).  Stops on the aggregate ||R||_F / ||B||_F.
    With dtype=float32 every workspace and every reduction is single
    precision (the fp32 emulation used to size test tolerances).
    """
    B = np.ascontiguousarray(B, dtype=dtype)
    dim, ncol = B.shape
    minv = np.asarray(minv, dtype=dtype)
    if minv.ndim == 1:
        minv = minv[:, None]
    X = np.zeros_like(B)
    bnorm = np.sqrt((B.astype(np.float64) ** 2).sum()) if dtype == np.float32 else np.linalg.norm(B)
    none = np.empty(0, dtype=np.int64)
    if bnorm == 0.0:
        return CgReport(X, 0, 0.0, True, none)
    if 1.0 <= cfg.tolerance:  # cg.py:121-122, X = 0 gives delta = 1
        return CgReport(X, 0, 1.0, True, none)

    R = B.copy()
    P = np.zeros_like(B)
    rho = np.ones(ncol, dtype=dtype)
    frozen = np.zeros(ncol, dtype=bool)

    def direction():
        # kernels.py:38-49: W = M^-1 R, eta = rho_new/rho (0 if rho == 0),
        # P = W + eta P (or R + eta P for the printed recursion)
        nonlocal P, rho
        W = R * minv
        rho_new = np.einsum("jq,jq->q", R, W)
        eta = _safe_ratio(rho_new, rho)
        P = P * eta + (R if cfg.printed_recursion else W)
        rho = rho_new

    direction()  # cg.py:133-135: the P = 0, rho = 1 pass initialises W, rho, P
    delta = 1.0
    steps = 0
    for u in range(1, cfg.max_steps + 1):
        psi = np.ascontiguousarray(apply_fn(P), dtype=dtype)
        # kernels.py:27-35
        pi = np.einsum("jq,jq->q", P, psi)
        gamma = _safe_ratio(rho, pi)
        X += P * gamma
        R -= psi * gamma
        rn2 = np.einsum("jq,jq->q", R, R)
        steps = u
        frozen |= pi == 0.0
        delta = float(np.sqrt(rn2.astype(np.float64).sum()) / bnorm)
        if not np.isfinite(delta):
            raise DivergenceError(u)
        if delta <= cfg.tolerance:
            break
        if u < cfg.max_steps:
            direction()
    return CgReport(X, steps, delta, delta <= cfg.tolerance, np.flatnonzero(frozen))


# ----------------------------------------------------------------------------
# CoFEM loop (cofem.py)

PROBE_STREAM = 3  # cofem.py:25


@dataclass(frozen=True)
class CofemConfig:
    """cofem.py:30-47."""

    iterations: int = 50
    probes: int = 20
    cg: CgConfig = field(default_factory=CgConfig)
    seed: int = 0
    variant: str = "standard"
    filter_percentile: float = 0.05
    clamp_max: float = 1e12
    floor_eps: float = 1e-12


def e_step(op, y, beta, alpha, cfg, rng=None, probes=None, dtype=np.float64):
    """cofem.py:76-100 -- solve A X = [P | Phi^T y]; mu = beta x_K, s from probes."""
    if probes is None:
        probes = draw_rademacher(op.n_cols, cfg.probes, rng)
    rhs = np.concatenate([probes, op.adjoint(np.asarray(y, dtype=np.float64)[:, None])], axis=1)
    minv = 1.0 / make_preconditioner(cfg.cg.theta_policy, op, beta, alpha)
    if dtype == np.float32:
        def apply_fn(V):
            return system_apply(op, beta, alpha, V.astype(np.float64)).astype(np.float32)
    else:
        def apply_fn(V):
            return system_apply(op, beta, alpha, V)
    rep = pcg_solve(apply_fn, rhs, minv, cfg.cg, dtype=dtype)
    sol = rep.solution.astype(np.float64)
    mu = beta * sol[:, cfg.probes]
    s = estimate_diagonal_rademacher(probes, sol[:, : cfg.probes])
    return mu, s, rep, probes


def m_step(mu, s, floor_eps=1e-12, clamp_max=1e12):
    """cofem.py:103-107 -- alpha = min(1 / max(mu^2 + s, floor), clamp)."""
    return np.minimum(1.0 / np.maximum(mu * mu + s, floor_eps), clamp_max)


def m_step_nonneg(mu, s, floor_eps=1e-12, clamp_max=1e12):
    """cofem.py:110-124 -- rectified second moment mu^2 + s + mu sqrt(s/pi)/erfcx(-xi)."""
    s = np.maximum(s, floor_eps)
    xi = mu / np.sqrt(2.0 * s)
    with np.errstate(over="ignore"):
        corr = mu * np.sqrt(s / np.pi) / erfcx(-xi)
    second = mu * mu + s + corr
    return np.minimum(1.0 / np.maximum(second, floor_eps), clamp_max)


def run_cofem(op, y, beta, cfg, probes_seq=None, dtype=np.float64):
    """cofem.py:136-157 -- T E-steps, M-step skipped after the last one.

    Returns (alpha, mu, s, diagnostics).  Probes come from substream(seed, 3)
    unless `probes_seq` (a list of D x K arrays, one per iteration) is given.
    """
    rng = substream(cfg.seed, PROBE_STREAM)
    alpha = np.ones(op.n_cols)
    update = m_step_nonneg if cfg.variant == "nonneg" else m_step
    diag = []
    mu = s = None
    for t in range(1, cfg.iterations + 1):
        probes = probes_seq[t - 1] if probes_seq is not None else None
        try:
            mu, s, rep, _ = e_step(op, y, beta, alpha, cfg, rng=rng, probes=probes, dtype=dtype)
        except DivergenceError as err:
            raise DivergenceError(err.step, f"EM iteration {t}") from err
        if t < cfg.iterations:
            alpha = update(mu, s, cfg.floor_eps, cfg.clamp_max)
        diag.append({"iteration": t, "cg_steps": rep.steps_taken,
                     "cg_residual": rep.final_relative_residual})
    return alpha, mu, s, diag


def run_cofem_multitask(ops, ys, beta, cfg, share_probes=False):
    """cofem.py:160-214 -- shared alpha; all tasks in one lockstep PCG call."""
    rng = substream(cfg.seed, PROBE_STREAM)
    dim = ops[0].n_cols
    L = len(ops)
    alpha = np.ones(dim)
    diag = []
    ests = None
    Q = cfg.probes + 1
    for t in range(1, cfg.iterations + 1):
        if share_probes:
            shared = draw_rademacher(dim, cfg.probes, rng)
            blocks = [shared] * L
        else:
            blocks = [draw_rademacher(dim, cfg.probes, rng) for _ in range(L)]
        rhs = np.concatenate(
            [np.concatenate([pb, op.adjoint(np.asarray(y, dtype=np.float64)[:, None])], axis=1)
             for op, y, pb in zip(ops, ys, blocks)], axis=1)
        minv = np.stack([1.0 / make_preconditioner(cfg.cg.theta_policy, op, beta, alpha)
                         for op in ops], axis=1)
        minv_cols = np.repeat(minv, Q, axis=1)

        def apply_fn(V):
            return np.concatenate([system_apply(op, beta, alpha, V[:, g * Q:(g + 1) * Q])
                                   for g, op in enumerate(ops)], axis=1)

        try:
            rep = pcg_solve(apply_fn, rhs, minv_cols, cfg.cg)
        except DivergenceError as err:
            raise DivergenceError(err.step, f"EM iteration {t}") from err
        ests = []
        for g, pb in enumerate(blocks):
            blk = rep.solution[:, g * Q:(g + 1) * Q]
            ests.append((beta * blk[:, cfg.probes], estimate_diagonal_rademacher(pb, blk[:, :cfg.probes])))
        if t < cfg.iterations:
            total = np.zeros(dim)
            for mu, s in ests:
                total = total + (mu ** 2 + s)
            alpha = np.minimum(L / np.maximum(total, cfg.floor_eps), cfg.clamp_max)
        diag.append({"iteration": t, "cg_steps": rep.steps_taken,
                     "cg_residual": rep.final_relative_residual})
    return alpha, ests, diag


def ozaki_dictionary(phi, bits=30):
    """The dictionary the 'ozaki' device mode multiplies (NOT reference code):
    Phi_ij rounded to round(Phi_ij / (r_i c_j) 2^30) r_i c_j / 2^30 (bits=30;
    'ozaki24' keeps three digit planes: bits=22) with
    power-of-two row scales r_i = 2^ceil(log2 max_j |Phi_ij|) and column
    scales c_j = 2^ceil(log2 max_i |Phi_ij| / r_i) (csrc/ozaki.cuh
    k_phi_rowscale / k_phi_colscale / k_phi_planes).  Running the reference
    recursion on this matrix separates representation sensitivity of a
    workload from kernel error."""
    phi = np.asarray(phi, dtype=np.float64)

    def p2(m):
        e = np.ceil(np.log2(np.where(m > 0, m, 1.0)))
        return np.where(m > 0, 2.0 ** e, 1.0)

    r = p2(np.abs(phi).max(axis=1))
    c = p2((np.abs(phi) / r[:, None]).max(axis=0))
    sc = r[:, None] * c[None, :]
    return np.rint(phi / sc * 2.0**bits) * sc / 2.0**bits


def ozaki_op(phi, bits=30):
    """Arithmetic model of the 'ozaki' device contraction (NOT reference code):
    the dictionary is ozaki_dictionary(phi); every operand column is rounded
    to 31-bit fixed point against its own power-of-two scale s_q =
    2^ceil(log2 max_j |M_jq w_j|) (w = Phi's column scales c for Phi V, its
    row scales r for Phi^T U; csrc/ozaki.cuh k_quantize / col_scale) and the
    int8 digit products are summed exactly, so the device result is this
    matrix product up to the final fp64 rounding.  Running the reference
    recursion with it reproduces the device's CG trajectory."""
    phi = np.asarray(phi, dtype=np.float64)

    def p2(m):
        return np.where(m > 0, 2.0 ** np.ceil(np.log2(np.where(m > 0, m, 1.0))), 1.0)

    r = p2(np.abs(phi).max(axis=1))
    c = p2((np.abs(phi) / r[:, None]).max(axis=0))
    phq = ozaki_dictionary(phi, bits)

    def qcols(M, w):
        X = M * w[:, None]
        s = p2(np.abs(X).max(axis=0))
        return np.rint(X / s * 2.0**30) * s / 2.0**30 / w[:, None]

    base = dense_op(phq)
    return Op(base.n_rows, base.n_cols, lambda V: phq @ qcols(V, c), lambda U: phq.T @ qcols(U, r),
              base.col_sq_norms, base.materialize, "dense")
