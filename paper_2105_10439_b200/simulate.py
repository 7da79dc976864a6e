"""Synthetic workloads of BASELINE.json (seeded stand-ins for the paper's data).

Stream layout follows the reference's simulate.build_problem
(/root/reference/pkg/src/sbl/simulate.py:242-249): dictionary from
substream(seed, 0), spikes from substream(seed, 1), noise from
substream(seed, 2); probes come from substream(seed, 3) inside run_cofem.
The dense dictionary is drawn float32 (N(0,1) scaled by 1/sqrt(N)) so the
GPU copy is exact; spike amplitudes are N(0, 1) as BASELINE.json specifies.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .cg import CgConfig
from .cofem import CofemConfig
from .operators import DenseOperator
from .problem import SblProblem, substream


@dataclass(frozen=True)
class DenseCsConfig:
    name: str
    N: int
    D: int
    frac: float      # fraction of nonzero coefficients
    sigma: float     # noise std; beta = 1 / sigma^2
    K: int           # probes
    T: int           # EM iterations
    U: int           # PCG step cap
    tol: float       # PCG tolerance
    seed: int = 0

    @property
    def beta(self):
        return 1.0 / self.sigma**2

    @property
    def n_spikes(self):
        return int(round(self.frac * self.D))

    def cofem_config(self, precision="ozaki", **over):
        cg = CgConfig(max_steps=self.U, tolerance=self.tol, precision=precision)
        kw = dict(iterations=self.T, probes=self.K, cg=cg, seed=self.seed)
        kw.update(over)
        return CofemConfig(**kw)


# BASELINE.json "configs" (dense Gaussian compressed sensing rows)
CONFIGS = {
    "dense-small": DenseCsConfig("dense-small", 256, 1024, 0.05, 0.01, 20, 50, 100, 1e-5),
    "dense-mid": DenseCsConfig("dense-mid", 4096, 16384, 0.02, 0.01, 20, 30, 200, 1e-5),
    "dense-large": DenseCsConfig("dense-large", 16384, 65536, 0.01, 0.01, 20, 20, 200, 1e-5),
}


@dataclass(frozen=True)
class ConvConfig:
    """BASELINE config 3: calcium-imaging-style deconvolution (synthetic)."""

    name: str
    D: int           # N = D time samples
    ntaps: int       # h[t] = exp(-t / tau), t < ntaps, unit L2 norm
    tau: float
    p: float         # Bernoulli spike probability per sample (Exp(1) amplitudes)
    sigma: float
    K: int
    T: int
    U: int
    tol: float
    seed: int = 0

    @property
    def N(self):
        return self.D

    @property
    def beta(self):
        return 1.0 / self.sigma**2

    def taps(self):
        h = np.exp(-np.arange(self.ntaps, dtype=np.float64) / self.tau)
        return h / np.linalg.norm(h)

    def cofem_config(self, precision="ozaki", **over):
        cg = CgConfig(max_steps=self.U, tolerance=self.tol, precision=precision)
        kw = dict(iterations=self.T, probes=self.K, cg=cg, seed=self.seed)
        kw.update(over)
        return CofemConfig(**kw)


CONV_CONFIGS = {
    "conv-large": ConvConfig("conv-large", 2**22, 256, 20.0, 0.01, 0.05, 30, 30, 200, 1e-5),
    "conv-mid": ConvConfig("conv-mid", 2**16, 256, 20.0, 0.01, 0.05, 30, 5, 200, 1e-5),
}


def spike_train(D, p, seed):
    """Nonnegative spikes: Bernoulli(p) support, Exp(1) amplitudes, substream(seed, 1)."""
    rng = substream(seed, 1)
    support = rng.random(D) < p
    return np.where(support, rng.exponential(1.0, D), 0.0)


def conv_problem(cfg: ConvConfig):
    """(SblProblem, z_true) for a convolution configuration; y computed in float64."""
    from scipy.signal import fftconvolve

    from .operators import ConvolutionOperator

    h = cfg.taps()
    z = spike_train(cfg.D, cfg.p, cfg.seed)
    y = fftconvolve(z, h)[: cfg.D] + cfg.sigma * substream(cfg.seed, 2).standard_normal(cfg.D)
    return SblProblem(y, ConvolutionOperator.from_taps(cfg.D, h), cfg.beta), z


@dataclass(frozen=True)
class Dct2Config:
    """BASELINE config 4: MRI-style undersampled 2-D DCT (synthetic)."""

    name: str
    n: int           # image side, D = n^2
    keep: float      # fraction of DCT coefficients kept (variable density)
    frac: float      # fraction of nonzero pixels, N(0,1) values
    sigma: float
    K: int
    T: int
    U: int
    tol: float
    seed: int = 0

    @property
    def D(self):
        return self.n * self.n

    @property
    def beta(self):
        return 1.0 / self.sigma**2

    def cofem_config(self, precision="ozaki", **over):
        cg = CgConfig(max_steps=self.U, tolerance=self.tol, precision=precision)
        kw = dict(iterations=self.T, probes=self.K, cg=cg, seed=self.seed)
        kw.update(over)
        return CofemConfig(**kw)


DCT_CONFIGS = {
    "dct-large": Dct2Config("dct-large", 1024, 0.25, 0.03, 0.01, 20, 20, 200, 1e-5),
    "dct-small": Dct2Config("dct-small", 128, 0.25, 0.03, 0.01, 20, 3, 200, 1e-5),
}


def dct2_problem(cfg: Dct2Config):
    """(SblProblem, z_true): mask from substream(seed, 0), pixels from
    substream(seed, 1), noise from substream(seed, 2); y in float64."""
    from scipy.fft import dctn

    from .operators import PartialDct2Operator, variable_density_mask

    mask = variable_density_mask(cfg.n, cfg.keep, substream(cfg.seed, 0))
    z = sparse_signal(cfg.D, int(round(cfg.frac * cfg.D)), cfg.seed)
    y = dctn(z.reshape(cfg.n, cfg.n), norm="ortho").ravel()[mask]
    y = y + cfg.sigma * substream(cfg.seed, 2).standard_normal(mask.size)
    return SblProblem(y, PartialDct2Operator(cfg.n, mask), cfg.beta), z


def gaussian_dictionary(N, D, seed):
    """N x D float32, entries N(0, 1/N), from substream(seed, 0)."""
    rng = substream(seed, 0)
    phi = rng.standard_normal((N, D), dtype=np.float32)
    phi *= np.float32(1.0 / np.sqrt(N))
    return phi


def sparse_signal(D, n_spikes, seed):
    """z with n_spikes uniformly placed N(0,1) entries, from substream(seed, 1)."""
    rng = substream(seed, 1)
    z = np.zeros(D)
    if n_spikes:
        support = rng.choice(D, size=n_spikes, replace=False)
        z[support] = rng.standard_normal(n_spikes)
    return z


def observe(phi, z, sigma, seed):
    """y = Phi z + sigma * N(0, I) in float64, noise from substream(seed, 2)."""
    nz = np.flatnonzero(z)
    y = phi[:, nz].astype(np.float64) @ z[nz]
    return y + sigma * substream(seed, 2).standard_normal(phi.shape[0])


def dense_cs_problem(cfg: DenseCsConfig, phi=None):
    """(SblProblem, z_true, phi) for a dense Gaussian CS configuration."""
    if phi is None:
        phi = gaussian_dictionary(cfg.N, cfg.D, cfg.seed)
    z = sparse_signal(cfg.D, cfg.n_spikes, cfg.seed)
    y = observe(phi, z, cfg.sigma, cfg.seed)
    return SblProblem(y, DenseOperator(phi, kind="dense-gaussian"), cfg.beta), z, phi


def nrmse(z_hat, z_true):
    """||zhat - z*|| / ||z*|| as a percentage (simulate.py:105-113)."""
    z_hat = np.asarray(z_hat, dtype=np.float64)
    z_true = np.asarray(z_true, dtype=np.float64)
    denom = np.linalg.norm(z_true)
    if denom == 0.0:
        raise ValueError("ground truth is identically zero")
    return 100.0 * np.linalg.norm(z_hat - z_true) / denom


def nmse(z_hat, z_true):
    """||zhat - z*||^2 / ||z*||^2 (the north_star's NMSE)."""
    return (nrmse(z_hat, z_true) / 100.0) ** 2
