"""GPU-resident dictionary operators and the implicit SBL system matrix.

Mirrors /root/reference/pkg/src/sbl/operators.py for the dense kind (the hot
path of this build): ``LinearOperator`` (:40-101), ``DenseOperator``
(:104-129), ``SystemMatrix`` (:248-272), ``build_dense_gaussian`` (:227-232)
and ``ShapeMismatchError`` (:21-27).

Every application runs on the GPU through the C ABI (include/cofem_b200.h).
A dictionary is stored once per precision mode: float32 matrices as given;
float64 matrices exactly (the "fp64" mode keeps the float64 entries in HBM,
the "ozaki" mode builds its 32-bit fixed-point digit planes from them).

Precision "auto" (the default of CgConfig) picks, per operator, the mode that
holds the reference's float64 results on that operator at the best speed:
float64 CUDA-core contractions where the dictionary is small enough that its
HBM stream does not matter (dense N*D <= 2^24 entries: <= 64 MB as float32,
L2-resident; short convolutions), the int8 tensor-core "ozaki" contractions
(float64-grade, 4 B/entry streamed) everywhere else, and the float64 FFT
passes for 2-D DCT dictionaries.
"""

from __future__ import annotations

import numpy as np

from . import _lib


class ShapeMismatchError(ValueError):
    """Input array shape is inconsistent with the operator (operators.py:21-27)."""

    def __init__(self, what, expected, actual):
        super().__init__(f"{what}: expected shape {expected}, got {actual}")
        self.expected = expected
        self.actual = actual


def _as_columns(V, nrows, what):
    V = np.asarray(V, dtype=np.float64)
    single = V.ndim == 1
    if single:
        V = V[:, None]
    if V.ndim != 2 or V.shape[0] != nrows:
        raise ShapeMismatchError(what, (nrows, "Q"), np.shape(V))
    return V, single


PRECISIONS = {"fp32": _lib.FP32, "fp64": _lib.FP64, "ozaki": _lib.OZAKI, "ozaki24": _lib.OZAKI24}
AUTO_FP64_ENTRIES = 1 << 24  # dense dictionaries up to this size run the float64 CUDA-core path under "auto"
AUTO_FP64_CONV_DIM = 1 << 16  # convolutions up to this length (and <= 512 taps) run the float64 FFT path


def check_precision(precision):
    if precision not in ("auto", "fp32", "fp64", "ozaki", "ozaki24"):
        raise ValueError("precision must be 'auto', 'fp32', 'fp64', 'ozaki' or 'ozaki24'")
    return precision


class LinearOperator:
    """An implicit N x D real matrix with apply / adjoint (operators.py:40-101)."""

    kind = "abstract"

    def __init__(self, n_rows, n_cols):
        if n_rows < 1 or n_cols < 1:
            raise ValueError(f"operator dims must be positive, got {n_rows} x {n_cols}")
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)

    def _apply(self, V):
        raise NotImplementedError

    def _apply_adjoint(self, U):
        raise NotImplementedError

    def apply(self, V):
        """Phi @ V for a (D,) vector or (D, Q) matrix."""
        V, single = _as_columns(V, self.n_cols, f"{self.kind} apply")
        out = self._apply(V)
        return out[:, 0] if single else out

    def apply_adjoint(self, U):
        """Phi^T @ U for an (N,) vector or (N, Q) matrix."""
        U, single = _as_columns(U, self.n_rows, f"{self.kind} apply_adjoint")
        out = self._apply_adjoint(U)
        return out[:, 0] if single else out

    def column_sq_norms(self):
        raise NotImplementedError

    def resolve_precision(self, precision):
        """The concrete device mode "auto" stands for on this operator."""
        return check_precision(precision)


class DenseOperator(LinearOperator):
    """Explicit dense dictionary, resident in HBM as float32 (operators.py:104-129).

    ``context(precision)`` returns the native context holding the matrix
    (created on first use; one per precision mode).
    """

    kind = "explicit-dense"

    def __init__(self, matrix, kind=None, device=0):
        matrix = np.array(matrix)
        if matrix.ndim != 2:
            raise ValueError("dense operator needs a 2-D matrix")
        super().__init__(*matrix.shape)
        if matrix.dtype != np.float32:
            matrix = matrix.astype(np.float64)
        matrix.flags.writeable = False
        self.matrix = matrix
        self.device = device
        if kind is not None:
            self.kind = kind
        self._ctx = {}

    def resolve_precision(self, precision):
        if check_precision(precision) != "auto":
            return precision
        # small: float64 CUDA-core contractions (L2-resident, exact); large: the
        # int8 tensor cores over the 24-bit fixed-point dictionary (3 B / entry:
        # the HBM stream is the bound; the reference's float64 run is matched
        # to ~3e-7 on BASELINE configs 2 and 3, tests/test_baseline_configs_gpu.py)
        return "fp64" if self.n_rows * self.n_cols <= AUTO_FP64_ENTRIES else "ozaki24"

    def context(self, precision="auto"):
        precision = self.resolve_precision(precision)
        code = PRECISIONS[precision]
        ctx = self._ctx.get(code)
        if ctx is None:
            ctx = self._ctx[code] = self.new_context(precision)
        return ctx

    def new_context(self, precision="auto"):
        """An uncached device copy (the caller closes it)."""
        precision = self.resolve_precision(precision)
        ctx = _lib.Context(self.n_rows, self.n_cols, PRECISIONS[precision], self.device)
        if self.matrix.dtype == np.float64:
            ctx.set_dictionary_f64(self.matrix)  # ozaki planes from the exact float64 entries
        else:
            ctx.set_dictionary(self.matrix)
        return ctx

    def release(self):
        """Free the device copies of the dictionary."""
        for ctx in self._ctx.values():
            ctx.close()
        self._ctx.clear()

    def apply_context(self):
        """The context plain applications use: float64 CUDA-core contractions,
        except that a large dictionary already resident in another mode (e.g.
        the "ozaki" planes of a run_cofem) is reused rather than uploaded a
        second time (its contraction error is ~2e-9)."""
        if self.n_rows * self.n_cols > AUTO_FP64_ENTRIES and self._ctx and PRECISIONS["fp64"] not in self._ctx:
            return next(iter(self._ctx.values()))
        return self.context("fp64")

    def _apply(self, V):
        return self.apply_context().apply(V)

    def _apply_adjoint(self, U):
        return self.apply_context().apply_adjoint(U)

    def materialize(self):
        return np.array(self.matrix, dtype=np.float64)

    def column_sq_norms(self):
        return self.apply_context().column_sq_norms()


MATERIALIZE_DCT_MAX = 8192  # SubsampledDctOperator: dims up to this run as a materialised dense dictionary


def _dct_mask(dim, mask):
    mask = np.asarray(mask, dtype=np.int64)
    if mask.ndim != 1 or mask.size < 1:
        raise ValueError("mask must be a nonempty 1-D index array")
    if np.unique(mask).size != mask.size:
        raise ValueError("mask indices must be distinct")
    if mask.min() < 0 or mask.max() >= dim:
        raise ValueError(f"mask indices must lie in [0, {dim})")
    mask = np.sort(mask)
    mask.flags.writeable = False
    return mask


def _dct1_column_sq_norms(dim, mask):
    """||Phi e_j||^2 = c_j^2 sum_i cos^2(pi (2 m_i + 1) j / 2D) (operators.py:165-179)
    = c_j^2 (N + Re(e^{i pi j / D} sum_i e^{2 pi i m_i j / D})) / 2: one FFT of
    the mask indicator instead of the reference's O(N D) cosine table."""
    scale = np.full(dim, 2.0 / dim)
    scale[0] = 1.0 / dim
    ind = np.zeros(dim)
    ind[mask] = 1.0
    j = np.arange(dim)
    s = np.real(np.exp(1j * np.pi * j / dim) * (dim * np.fft.ifft(ind)))
    return scale * (0.5 * mask.size + 0.5 * s)


class SubsampledDctOperator(DenseOperator):
    """Phi = M Omega^{-1}: inverse orthonormal DCT-II rows selected by a mask
    (operators.py:132-179).  Small dims (<= MATERIALIZE_DCT_MAX) are
    materialised once (float64, N x D) and run as a dense dictionary (exact
    float64 contractions under "auto"); larger ones -- or ``fast=True`` --
    construct a :class:`FastSubsampledDctOperator`, the O(D log D) device
    path (same interface, no N x D matrix)."""

    kind = "undersampled-dct"

    def __new__(cls, dim, mask, device=0, fast=None):
        if fast or (fast is None and dim > MATERIALIZE_DCT_MAX):
            return FastSubsampledDctOperator(dim, mask, device)
        return super().__new__(cls)

    def __init__(self, dim, mask, device=0, fast=None):
        from scipy.fft import idct

        mask = _dct_mask(dim, mask)
        super().__init__(idct(np.eye(dim), axis=0, norm="ortho")[mask, :], device=device)
        self.mask = mask

    def resolve_precision(self, precision):
        # exact float64 contractions: orthonormal-row DCT dictionaries make CG's
        # step count sensitive to any rounding of Phi
        return "fp64" if check_precision(precision) == "auto" else precision

    def column_sq_norms(self):
        """Analytic column norms, operators.py:165-179."""
        return _dct1_column_sq_norms(self.n_cols, self.mask)


class FastSubsampledDctOperator(LinearOperator):
    """The reference's SubsampledDctOperator (operators.py:132-179) without a
    materialised matrix, any D: on the GPU Phi V = DCT-III(V)[mask], Phi^T U =
    DCT-II(scatter(U)) and Phi^T Phi = DCT-II(mask .* DCT-III(.)), each a
    batched complex length-D FFT with Makhoul's packing of two real columns
    (csrc/dct1.cuh; cuFFT double complex for the FFTs themselves) -- O(D log D)
    per column instead of O(N D).  Float64 whatever the precision mode."""

    kind = "undersampled-dct"

    def __init__(self, dim, mask, device=0):
        mask = _dct_mask(dim, mask)
        super().__init__(mask.size, dim)
        self.mask = mask
        self.device = device
        self._ctx = {}

    def resolve_precision(self, precision):
        return "fp64" if check_precision(precision) == "auto" else precision

    def context(self, precision="auto"):
        precision = self.resolve_precision(precision)
        ctx = self._ctx.get("fft")
        if ctx is None:
            ctx = self._ctx["fft"] = self.new_context(precision)
        return ctx

    def apply_context(self):
        return self.context()

    def new_context(self, precision="auto"):
        precision = self.resolve_precision(precision)
        if precision == "fp32":
            raise NotImplementedError("1-D DCT dictionaries run the float64 FFT path")
        return _lib.Context.dct1(self.n_cols, self.mask, _lib.FP64, self.device)

    def release(self):
        for ctx in self._ctx.values():
            ctx.close()
        self._ctx.clear()

    def _apply(self, V):
        return self.context().apply(V)

    def _apply_adjoint(self, U):
        return self.context().apply_adjoint(U)

    def column_sq_norms(self):
        return _dct1_column_sq_norms(self.n_cols, self.mask)


def build_undersampled_dct(dim, n_rows, rng):
    """Orthonormal DCT-II rows subsampled uniformly without replacement (operators.py:235-240)."""
    if not 1 <= n_rows <= dim:
        raise ValueError(f"need 1 <= N <= D, got N={n_rows}, D={dim}")
    return SubsampledDctOperator(dim, rng.choice(dim, size=n_rows, replace=False))


class ConvolutionOperator(LinearOperator):
    """Causal convolution with a filter h: the D x D lower-triangular Toeplitz
    matrix Phi_ij = h[i - j] (operators.py:182-225).

    ``ConvolutionOperator(dim, decay)`` is the reference's filter
    h[m] = (1 - decay)^m, m < D; ``ConvolutionOperator.from_taps(dim, taps)``
    takes any FIR filter (BASELINE config 3: exp(-t/20), 256 taps, unit norm).
    On the GPU both Phi and Phi^T run as banded int8 tensor-core contractions
    (precision "ozaki"); taps below 2^-34 of the largest one are dropped there
    (they are under the 2^-30 fixed-point resolution of the band).
    """

    kind = "exp-convolution"

    def __init__(self, dim, decay=None, taps=None, device=0):
        super().__init__(dim, dim)
        if taps is None:
            if decay is None or not 0.0 < decay < 1.0:
                raise ValueError(f"decay must lie in (0, 1), got {decay}")
            self.decay = float(decay)
            taps = (1.0 - self.decay) ** np.arange(dim, dtype=np.float64)
        else:
            self.decay = None
            self.kind = "fir-convolution"
            taps = np.asarray(taps, dtype=np.float64)
            if taps.ndim != 1 or not 1 <= taps.size <= dim:
                raise ValueError("taps must be a 1-D array of length 1..dim")
        taps = np.array(taps, dtype=np.float64)
        taps.flags.writeable = False
        self.filter = taps
        self.device = device
        self._ctx = {}

    @classmethod
    def from_taps(cls, dim, taps, device=0):
        return cls(dim, taps=taps, device=device)

    def gpu_taps(self):
        h = self.filter
        keep = np.flatnonzero(np.abs(h) >= np.abs(h).max() * 2.0**-34)
        return h[: keep[-1] + 1] if keep.size else h[:1]

    def fft_taps(self):
        """The filter for the float64 FFT path: taps below 2^-60 of the largest
        one are dropped (far under float64 resolution)."""
        h = self.filter
        keep = np.flatnonzero(np.abs(h) >= np.abs(h).max() * 2.0**-60)
        return h[: keep[-1] + 1] if keep.size else h[:1]

    def resolve_precision(self, precision):
        if check_precision(precision) != "auto":
            return precision
        short = self.n_cols <= AUTO_FP64_CONV_DIM and self.fft_taps().size <= 512
        # long: the banded int8 tensor-core kernels with 24-bit taps (config 3 at
        # full size: mu / alpha within 2.3e-6 of the reference's float64 run)
        return "fp64" if short else "ozaki24"

    def context(self, precision="auto"):
        precision = self.resolve_precision(precision)
        ctx = self._ctx.get(precision)
        if ctx is None:
            ctx = self._ctx[precision] = self.new_context(precision)
        return ctx

    def new_context(self, precision="auto"):
        """'ozaki': banded int8 tensor-core kernel (any filter length; 32-bit
        fixed-point taps), 'ozaki24': the same with 24-bit taps (three band
        digit planes, a quarter fewer MMAs); 'fp64': float64 overlap-save FFT
        passes (filters up to 512 taps)."""
        precision = self.resolve_precision(precision)
        if precision in ("ozaki", "ozaki24"):
            code = _lib.OZAKI24 if precision == "ozaki24" else _lib.OZAKI
            return _lib.Context.convolution(self.n_cols, self.gpu_taps(), code, self.device)
        if precision == "fp64":
            return _lib.Context.convolution(self.n_cols, self.fft_taps(), _lib.FP64, self.device)
        raise NotImplementedError("convolution dictionaries run in the 'ozaki' or 'fp64' precision mode")

    def release(self):
        for ctx in self._ctx.values():
            ctx.close()
        self._ctx.clear()

    def _apply(self, V):
        return self.context().apply(V)

    def _apply_adjoint(self, U):
        return self.context().apply_adjoint(U)

    def apply_context(self):
        return self.context()

    def materialize(self):
        d, h = self.n_cols, self.filter
        m = np.zeros((d, d))
        for j in range(d):
            n = min(h.size, d - j)
            m[j:j + n, j] = h[:n]
        return m

    def column_sq_norms(self):
        """Truncated geometric / FIR sums: column j holds h[0 : min(L, D - j)]."""
        c = np.concatenate([[0.0], np.cumsum(self.filter * self.filter)])
        return c[np.minimum(self.filter.size, self.n_cols - np.arange(self.n_cols))]


class PartialDct2Operator(LinearOperator):
    """Row subset of the orthonormal 2-D DCT-II of n x n images (BASELINE config 4;
    the 2-D analogue of the reference's SubsampledDctOperator, operators.py:132-179).

    z is an n x n image flattened row-major (D = n^2); Phi z = the coefficients
    at the flat indices ``mask`` (k n + l, sorted, distinct) of
    ``scipy.fft.dctn(z, norm="ortho")``.  Rows are orthonormal (Phi Phi^T = I).
    On the GPU Phi^T Phi is three fused float64 FFT passes (row DCT-II, column
    DCT-II / mask / DCT-III, row DCT-III + PCG combine); n a power of two in
    [64, 1024].  Precision "ozaki" and "fp64" both select this float64 path.
    """

    kind = "partial-dct2"

    def __init__(self, n, mask, device=0):
        mask = np.asarray(mask, dtype=np.int64)
        if mask.ndim != 1 or mask.size < 1:
            raise ValueError("mask must be a nonempty 1-D index array")
        if np.unique(mask).size != mask.size:
            raise ValueError("mask indices must be distinct")
        if mask.min() < 0 or mask.max() >= n * n:
            raise ValueError(f"mask indices must lie in [0, {n * n})")
        super().__init__(mask.size, n * n)
        mask = np.sort(mask)
        mask.flags.writeable = False
        self.n = int(n)
        self.mask = mask
        self.device = device
        self._ctx = {}

    def resolve_precision(self, precision):
        return "fp64" if check_precision(precision) == "auto" else precision

    def context(self, precision="auto"):
        precision = self.resolve_precision(precision)
        ctx = self._ctx.get("fft")
        if ctx is None:
            ctx = self._ctx["fft"] = self.new_context(precision)
        return ctx

    def apply_context(self):
        return self.context()

    def new_context(self, precision="auto"):
        precision = self.resolve_precision(precision)
        if precision not in ("ozaki", "ozaki24", "fp64"):
            raise NotImplementedError("2-D DCT dictionaries run the float64 FFT path ('ozaki' or 'fp64')")
        return _lib.Context.dct2(self.n, self.mask, _lib.FP64, self.device)

    def release(self):
        for ctx in self._ctx.values():
            ctx.close()
        self._ctx.clear()

    def _apply(self, V):
        return self.context().apply(V)

    def _apply_adjoint(self, U):
        return self.context().apply_adjoint(U)

    def dct_matrix(self):
        n = self.n
        k = np.arange(n)[:, None]
        i = np.arange(n)[None, :]
        c = np.cos(np.pi * (2 * i + 1) * k / (2.0 * n))
        c *= np.where(k == 0, np.sqrt(1.0 / n), np.sqrt(2.0 / n))
        return c

    def column_sq_norms(self):
        """||Phi e_ij||^2 = sum_{(k,l) in mask} C_ki^2 C_lj^2 = ((C.C)^T M (C.C))_ij."""
        c2 = self.dct_matrix() ** 2
        grid = np.zeros(self.n * self.n)
        grid[self.mask] = 1.0
        return (c2.T @ grid.reshape(self.n, self.n) @ c2).ravel()


def variable_density_mask(n, keep_frac, rng, r0=None):
    """MRI-style mask: keep probability ~ 1/(1 + r/r0)^2 (r = radius from the DC
    coefficient, r0 = 64 at n = 1024), normalised so the expected kept fraction
    is keep_frac; one Bernoulli draw per coefficient."""
    r0 = 64.0 * n / 1024.0 if r0 is None else r0
    k = np.arange(n)
    r = np.sqrt(k[:, None] ** 2 + k[None, :] ** 2)
    w = 1.0 / (1.0 + r / r0) ** 2
    target = keep_frac * n * n
    lo, hi = 0.0, 1.0 / w.min()
    for _ in range(100):  # bisection for c: sum min(1, c w) = target
        mid = 0.5 * (lo + hi)
        if np.minimum(1.0, mid * w).sum() < target:
            lo = mid
        else:
            hi = mid
    p = np.minimum(1.0, hi * w)
    return np.flatnonzero(rng.random(n * n) < p.ravel())


def build_exp_convolution(dim, decay):
    """Lower-triangular convolution with filter (1-rho)^m, m = 0..D-1 (operators.py:243-245)."""
    return ConvolutionOperator(dim, decay)


def build_dense_gaussian(n_rows, dim, rng, dtype=np.float64):
    """Dense dictionary with i.i.d. N(0, 1/N) entries (operators.py:227-232).

    The default draw is the reference's (``rng.normal(0, 1/sqrt(N))`` in
    float64, same generator consumption), held exactly on the device.
    ``dtype=np.float32`` draws ``rng.standard_normal(dtype=float32)`` instead:
    a float32-exact dictionary at half the host memory and upload (a
    different draw from the same seed).
    """
    if not 1 <= n_rows <= dim:
        raise ValueError(f"need 1 <= N <= D, got N={n_rows}, D={dim}")
    if np.dtype(dtype) == np.float32:
        entries = rng.standard_normal((n_rows, dim), dtype=np.float32) * np.float32(1.0 / np.sqrt(n_rows))
    else:
        entries = rng.normal(0.0, 1.0 / np.sqrt(n_rows), size=(n_rows, dim))
    return DenseOperator(entries, kind="dense-gaussian")


class SystemMatrix:
    """Implicit A = beta Phi^T Phi + diag(alpha), SPD by construction (operators.py:248-272)."""

    def __init__(self, op, beta, alpha):
        if beta <= 0:
            raise ValueError(f"beta must be positive, got {beta}")
        alpha = np.array(alpha, dtype=np.float64)
        if alpha.shape != (op.n_cols,):
            raise ShapeMismatchError("alpha", (op.n_cols,), alpha.shape)
        if not np.all(alpha > 0):
            raise ValueError("alpha entries must all be positive")
        alpha.flags.writeable = False
        self.op = op
        self.beta = float(beta)
        self.alpha = alpha

    @property
    def dim(self):
        return self.op.n_cols

    def apply(self, V, precision=None):
        """A @ V on the GPU without materialising A (the operator's apply
        context unless a precision mode is named)."""
        V, single = _as_columns(V, self.dim, "system apply")
        ctx = self.op.apply_context() if precision is None else self.op.context(precision)
        out = ctx.system_apply(self.beta, self.alpha, V)
        return out[:, 0] if single else out
