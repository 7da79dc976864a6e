"""Golden runs of the REAL reference at BASELINE.json's full sizes (build container only).

    SBL_BACKEND=numpy python tests/golden/make_golden_large.py dense-large
    SBL_BACKEND=numpy python tests/golden/make_golden_large.py dense-mid30
    SBL_BACKEND=numpy python tests/golden/make_golden_large.py dct-large
    SBL_BACKEND=numpy python tests/golden/make_golden_large.py conv-large

Each target runs the reference's own `run_cofem` (/root/reference/pkg/src/sbl/
cofem.py:136-157, float64 numpy) on the seeded synthetic problem the GPU tests
rebuild on the box from the same seeds (paper_2105_10439_b200/simulate.py).
The two structured configs have no operator class in the reference, so they
are given to the reference's CoFEM loop as subclasses of the reference's own
`LinearOperator` (operators.py:40-101) with the semantics BASELINE.json
states: causal Toeplitz convolution with a 256-tap truncated filter (the
truncated form of operators.py:182-225) and row-subsampled orthonormal 2-D
DCT-II (the 2-D form of operators.py:132-179).

Storage: the dense configs keep the whole mu / alpha / s; the 2^20 / 2^22
configs keep a fixed random sample of 65536 coordinates, the support
(alpha < 1e6, test_cofem.py:347) as a bit mask, the full-vector norms and
block sums, and the per-iteration CG steps and residuals.  The dictionaries
themselves are regenerated from their seeds and checked by digest.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)
os.environ.setdefault("SBL_BACKEND", "numpy")

import sbl  # noqa: E402  (the reference)
from sbl import cofem as ref_cofem  # noqa: E402
from sbl.operators import DenseOperator, LinearOperator  # noqa: E402
from sbl.problem import SblProblem  # noqa: E402

from paper_2105_10439_b200 import simulate as S  # noqa: E402  (problem generators only)

SAMPLE = 65536
BLOCKS = 1024


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def sample_index(D):
    return np.sort(np.random.default_rng(20261020).choice(D, size=min(SAMPLE, D), replace=False))


class TruncatedConvolution(LinearOperator):
    """Causal D x D Toeplitz convolution with a short filter `taps`; FFT path
    zero-padded to >= D + L - 1 like operators.py:200-211."""

    kind = "truncated-convolution"

    def __init__(self, dim, taps):
        from scipy.fft import next_fast_len, rfft

        super().__init__(dim, dim)
        self.taps = np.asarray(taps, dtype=np.float64)
        self._pad = next_fast_len(dim + self.taps.size - 1)
        self._spec = rfft(self.taps, self._pad)

    def _apply(self, V):
        from scipy.fft import irfft, rfft

        return irfft(rfft(V, self._pad, axis=0) * self._spec[:, None], self._pad, axis=0)[: self.n_rows]

    def _apply_adjoint(self, U):
        from scipy.fft import irfft, rfft

        return irfft(rfft(U, self._pad, axis=0) * np.conj(self._spec)[:, None], self._pad, axis=0)[: self.n_cols]

    def column_sq_norms(self):
        c = np.concatenate([[0.0], np.cumsum(self.taps**2)])
        return c[np.minimum(self.taps.size, self.n_cols - np.arange(self.n_cols))]


class PartialDct2(LinearOperator):
    """Rows `mask` of the orthonormal 2-D DCT-II of n x n images (row-major)."""

    kind = "partial-dct2"

    def __init__(self, n, mask):
        super().__init__(len(mask), n * n)
        self.n = n
        self.mask = np.sort(np.asarray(mask, dtype=np.int64))

    def _apply(self, V):
        from scipy.fft import dctn

        n, q = self.n, V.shape[1]
        return dctn(V.reshape(n, n, q), axes=(0, 1), norm="ortho").reshape(n * n, q)[self.mask]

    def _apply_adjoint(self, U):
        from scipy.fft import idctn

        n, q = self.n, U.shape[1]
        full = np.zeros((n * n, q))
        full[self.mask] = U
        return idctn(full.reshape(n, n, q), axes=(0, 1), norm="ortho").reshape(n * n, q)


def _run(problem, cfg, tag):
    t0 = time.time()
    state, est, diag = ref_cofem.run_cofem(problem, cfg)
    steps = [r["cg_steps"] for r in diag]
    print(f"{tag}: {time.time() - t0:.0f} s, steps {steps}", flush=True)
    return state, est, diag


def _common(state, est, diag, z):
    return dict(
        cg_steps=np.array([r["cg_steps"] for r in diag]),
        cg_residuals=np.array([r["cg_residual"] for r in diag]),
        wall_time=np.array([r["wall_time"] for r in diag]),
        nmse=np.array(S.nmse(est.mu, z)),
        z_digest=np.array(digest(z)),
    )


def make_dense(name, iterations, fname):
    c = S.CONFIGS[name]
    phi = S.gaussian_dictionary(c.N, c.D, c.seed)
    z = S.sparse_signal(c.D, c.n_spikes, c.seed)
    y = S.observe(phi, z, c.sigma, c.seed)
    print(f"{name}: phi {phi.shape} digest {digest(phi)}", flush=True)
    op = DenseOperator(phi.astype(np.float64))
    del phi
    cfg = sbl.CofemConfig(iterations=iterations, probes=c.K, seed=c.seed,
                          cg=sbl.CgConfig(max_steps=c.U, tolerance=c.tol))
    state, est, diag = _run(SblProblem(y, op, c.beta), cfg, name)
    np.savez_compressed(
        os.path.join(HERE, fname),
        config=np.array([c.N, c.D, c.K, iterations, c.U, c.tol, c.beta, c.seed, c.frac, c.sigma]),
        phi_digest=np.array(digest(S.gaussian_dictionary(c.N, c.D, c.seed))),
        y=y, alpha=state.alpha, mu=est.mu, s=est.s, **_common(state, est, diag, z))


def _save_sampled(fname, cfgrow, y, z, state, est, diag, extra):
    D = est.mu.size
    idx = sample_index(D)
    alpha = state.alpha
    np.savez_compressed(
        os.path.join(HERE, fname),
        config=np.array(cfgrow),
        y_digest=np.array(digest(y)),
        sample=idx.astype(np.int32),
        mu_sample=est.mu[idx], alpha_sample=alpha[idx], s_sample=est.s[idx],
        support_bits=np.packbits(alpha < 1e6),
        norms=np.array([np.linalg.norm(est.mu), np.linalg.norm(alpha), np.linalg.norm(est.s)]),
        mu_blocks=est.mu.reshape(BLOCKS, -1).sum(axis=1),
        s_blocks=est.s.reshape(BLOCKS, -1).sum(axis=1),
        loga_blocks=np.log(alpha).reshape(BLOCKS, -1).sum(axis=1),
        **_common(state, est, diag, z), **extra)


def make_dct(iterations):
    from scipy.fft import dctn

    from paper_2105_10439_b200.operators import variable_density_mask
    from paper_2105_10439_b200.problem import substream

    c = S.DCT_CONFIGS["dct-large"]
    mask = variable_density_mask(c.n, c.keep, substream(c.seed, 0))
    z = S.sparse_signal(c.D, int(round(c.frac * c.D)), c.seed)
    y = dctn(z.reshape(c.n, c.n), norm="ortho").ravel()[mask]
    y = y + c.sigma * substream(c.seed, 2).standard_normal(mask.size)
    cfg = sbl.CofemConfig(iterations=iterations, probes=c.K, seed=c.seed,
                          cg=sbl.CgConfig(max_steps=c.U, tolerance=c.tol))
    state, est, diag = _run(SblProblem(y, PartialDct2(c.n, mask), c.beta), cfg, "dct-large")
    _save_sampled(f"cofem_dct-large_T{iterations}.npz",
                  [c.n, c.D, c.K, iterations, c.U, c.tol, c.beta, c.seed, c.frac, c.sigma, c.keep],
                  y, z, state, est, diag, dict(mask_digest=np.array(digest(mask))))


def make_conv(iterations):
    from scipy.signal import fftconvolve

    from paper_2105_10439_b200.problem import substream

    c = S.CONV_CONFIGS["conv-large"]
    h = c.taps()
    z = S.spike_train(c.D, c.p, c.seed)
    y = fftconvolve(z, h)[: c.D] + c.sigma * substream(c.seed, 2).standard_normal(c.D)
    cfg = sbl.CofemConfig(iterations=iterations, probes=c.K, seed=c.seed,
                          cg=sbl.CgConfig(max_steps=c.U, tolerance=c.tol))
    state, est, diag = _run(SblProblem(y, TruncatedConvolution(c.D, h), c.beta), cfg, "conv-large")
    _save_sampled(f"cofem_conv-large_T{iterations}.npz",
                  [c.D, c.ntaps, c.tau, c.K, iterations, c.U, c.tol, c.beta, c.seed, c.p, c.sigma],
                  y, z, state, est, diag, {})


if __name__ == "__main__":
    which = sys.argv[1]
    T = int(sys.argv[2]) if len(sys.argv) > 2 else None
    if which == "dense-large":
        make_dense("dense-large", T or 20, f"cofem_dense-large_T{T or 20}.npz")
    elif which == "dense-mid30":
        make_dense("dense-mid", 30, "cofem_dense-mid_T30.npz")
    elif which == "dct-large":
        make_dct(T or 20)
    elif which == "conv-large":
        make_conv(T or 2)
    else:
        raise SystemExit(f"unknown target {which}")
