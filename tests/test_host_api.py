"""Host-side logic of the drop-in API (no GPU): validation, probe streams,
preconditioner construction, generators.  Mirrors the validation cases of the
reference's tests (test_cg.py, test_cofem.py, test_operators.py)."""

import numpy as np
import pytest

from oracle import cofem_oracle as O
from paper_2105_10439_b200 import (
    CgConfig,
    CofemConfig,
    DenseOperator,
    PosteriorEstimate,
    Preconditioner,
    PrecisionState,
    SblProblem,
    ShapeMismatchError,
    SystemMatrix,
    draw_probe_blocks,
    draw_rademacher,
    estimate_diagonal_rademacher,
    m_step,
    m_step_nonneg,
    make_preconditioner,
    substream,
)
from paper_2105_10439_b200 import simulate as S
from paper_2105_10439_b200.probes import draw_rademacher_int8


def test_config_validation():
    with pytest.raises(ValueError):
        CgConfig(max_steps=0)
    with pytest.raises(ValueError):
        CgConfig(tolerance=0.0)
    with pytest.raises(ValueError):
        CgConfig(precision="fp16")
    with pytest.raises(ValueError, match="iterations"):
        CofemConfig(iterations=0)
    with pytest.raises(ValueError, match="variant"):
        CofemConfig(variant="laplace")
    with pytest.raises(ValueError, match="filter_percentile"):
        CofemConfig(filter_percentile=1.5)


def test_preconditioner_validation_and_policies():
    with pytest.raises(ValueError):
        Preconditioner(m=np.array([1.0, 0.0]))
    np.testing.assert_array_equal(Preconditioner.identity(3).m, np.ones(3))
    op = DenseOperator(np.zeros((4, 5)))
    np.testing.assert_array_equal(make_preconditioner("all-ones", op, 1e4, np.ones(5)).m, np.full(5, 10001.0))
    np.testing.assert_array_equal(make_preconditioner("none", op, 1e4, np.ones(5)).m, np.ones(5))
    custom = make_preconditioner(np.arange(1.0, 6.0), op, 2.0, np.ones(5))
    np.testing.assert_array_equal(custom.m, 2.0 * np.arange(1.0, 6.0) + 1.0)
    with pytest.raises(ValueError, match="custom theta"):
        make_preconditioner(np.array([1.0, -2.0, 3.0, 4.0, 5.0]), op, 2.0, np.ones(5))
    with pytest.raises(ValueError, match="theta policy"):
        make_preconditioner("spectral", op, 2.0, np.ones(5))
    with pytest.raises(ValueError, match="alpha"):
        make_preconditioner("all-ones", op, 2.0, np.zeros(5))


def test_system_and_problem_validation():
    op = DenseOperator(np.eye(4))
    with pytest.raises(ValueError, match="beta"):
        SystemMatrix(op, 0.0, np.ones(4))
    with pytest.raises(ShapeMismatchError):
        SystemMatrix(op, 1.0, np.ones(5))
    with pytest.raises(ValueError, match="alpha"):
        SystemMatrix(op, 1.0, np.array([1.0, 1.0, 0.0, 1.0]))
    with pytest.raises(ShapeMismatchError):
        SblProblem(np.ones(3), op, 1.0)
    with pytest.raises(ValueError, match="beta"):
        SblProblem(np.ones(4), op, -1.0)
    with pytest.raises(ValueError):
        DenseOperator(np.empty((0, 3)))
    dense = DenseOperator(np.ones((2, 3)))
    with pytest.raises(ValueError):
        dense.matrix[0, 0] = 2.0


def test_probe_stream_matches_reference_draws():
    # the int8 draw consumes the generator exactly like probes.py:13-17
    a = draw_rademacher_int8(257, 9, substream(7, 3))
    b = O.draw_rademacher(257, 9, substream(7, 3))
    np.testing.assert_array_equal(a.astype(np.float64), b)
    np.testing.assert_array_equal(draw_rademacher(257, 9, substream(7, 3)), b)
    # T sequential blocks, as run_cofem draws them (cofem.py:143-151)
    blocks = draw_probe_blocks(64, 5, 4, seed=11)
    rng = substream(11, 3)
    for t in range(4):
        np.testing.assert_array_equal(blocks[t].astype(np.float64), O.draw_rademacher(64, 5, rng))
    with pytest.raises(ValueError):
        draw_rademacher(0, 3, substream(0, 0))


def test_estimator_and_m_steps_match_oracle(rng):
    probes = draw_rademacher(12, 7, rng)
    np.testing.assert_array_equal(estimate_diagonal_rademacher(probes, probes), np.ones(12))
    X = rng.standard_normal((12, 7))
    np.testing.assert_allclose(estimate_diagonal_rademacher(probes, X),
                               O.estimate_diagonal_rademacher(probes, X), rtol=1e-15)
    state = PrecisionState.initial(2)
    upd = m_step(PosteriorEstimate(mu=np.array([1.0, 0.0]), s=np.array([0.0, -1.0])), state)
    np.testing.assert_array_equal(upd.alpha, [1.0, state.clamp_max])
    assert upd.iteration == 2
    mu = rng.standard_normal(50) * 3
    s = rng.random(50) - 0.2
    np.testing.assert_allclose(m_step_nonneg(PosteriorEstimate(mu, s), PrecisionState.initial(50)).alpha,
                               O.m_step_nonneg(mu, s), rtol=1e-14)


def test_simulate_generators_are_deterministic():
    c = S.CONFIGS["dense-small"]
    p1, z1, phi1 = S.dense_cs_problem(c)
    p2, z2, phi2 = S.dense_cs_problem(c)
    np.testing.assert_array_equal(phi1, phi2)
    np.testing.assert_array_equal(np.asarray(p1.y), np.asarray(p2.y))
    assert phi1.dtype == np.float32 and phi1.shape == (c.N, c.D)
    assert np.count_nonzero(z1) == c.n_spikes
    assert 0.8 / c.N <= phi1.astype(np.float64).var() <= 1.2 / c.N
    assert p1.beta == pytest.approx(1e4)
    assert S.nrmse(z1, z1) == 0.0


def test_dct2_oracle_and_mask_generator():
    from scipy.fft import dctn

    from paper_2105_10439_b200 import PartialDct2Operator, variable_density_mask

    rng = np.random.default_rng(4)
    n = 16
    mask = variable_density_mask(n, 0.25, substream(0, 0))
    again = variable_density_mask(n, 0.25, substream(0, 0))
    np.testing.assert_array_equal(mask, again)
    assert 0.1 < mask.size / n**2 < 0.4 and 0 in mask  # DC always kept
    op = O.dct2_op(n, mask)
    V = rng.standard_normal((n * n, 3))
    U = rng.standard_normal((mask.size, 3))
    np.testing.assert_allclose(op.apply(V)[:, 1], dctn(V[:, 1].reshape(n, n), norm="ortho").ravel()[mask])
    assert abs(np.sum(U * op.apply(V)) - np.sum(op.adjoint(U) * V)) < 1e-10
    np.testing.assert_allclose(op.apply(op.adjoint(U)), U, atol=1e-12)  # orthonormal rows
    m = op.materialize()
    np.testing.assert_allclose(op.col_sq_norms(), (m * m).sum(axis=0), atol=1e-12)
    np.testing.assert_allclose(PartialDct2Operator(n, mask).column_sq_norms(), op.col_sq_norms(), atol=1e-12)
    with pytest.raises(ValueError, match="distinct"):
        PartialDct2Operator(4, np.array([1, 1]))


def test_multitask_validation_before_any_device_work():
    from paper_2105_10439_b200 import MultiTaskProblem, run_cofem_multitask

    prob = SblProblem(np.ones(4), DenseOperator(np.ones((4, 8))), 1e4)
    with pytest.raises(ValueError, match="standard"):
        run_cofem_multitask(MultiTaskProblem((prob,)), CofemConfig(variant="nonneg"))
    with pytest.raises(ShapeMismatchError):
        MultiTaskProblem((prob, SblProblem(np.ones(4), DenseOperator(np.ones((4, 9))), 1e4)))


def test_dct_step_sensitivity_is_a_reference_property():
    """The reference recursion (oracle, bit-exact with it) on the undersampled
    DCT workload of test_cofem.py:257-265 changes its CG step counts when Phi is
    rounded to the device's 32-bit fixed-point representation -- the basis of
    the step tolerance in test_gpu_parity.assert_dct_steps_close."""
    from scipy.fft import idct

    from conftest import golden

    g = golden("reference_workloads.npz")
    phi = idct(np.eye(1024), axis=0, norm="ortho")[np.sort(g["dct_mask"]), :]
    cfg = O.CofemConfig(iterations=3, probes=20, seed=0)
    _, _, _, exact = O.run_cofem(O.dense_op(phi), g["dct_y"], float(g["dct_beta"]), cfg)
    _, _, _, quant = O.run_cofem(O.dense_op(O.ozaki_dictionary(phi)), g["dct_y"], float(g["dct_beta"]), cfg)
    assert [d["cg_steps"] for d in exact] == list(g["dct_steps"][:3])
    assert [d["cg_steps"] for d in quant][1] > [d["cg_steps"] for d in exact][1]
    assert np.abs(O.ozaki_dictionary(phi) - phi).max() <= 2.0**-31


def _dct1_packed(D):
    """Makhoul's packed two-columns-per-complex-FFT DCT-II / DCT-III (the
    algorithm of csrc/dct1.cuh, numpy FFTs): exact, but rounded differently
    from scipy's dct / idct."""
    m = np.arange(D)
    sig = np.where(m < (D + 1) // 2, 2 * m, 2 * (D - 1 - m) + 1)
    k = np.arange(D)
    c = np.full(D, np.sqrt(2.0 / D))
    c[0] = np.sqrt(1.0 / D)
    tw = np.exp(-1j * np.pi * k / (2 * D))

    def dct2(a, b):
        Z = np.fft.fft(a[sig] + 1j * b[sig])
        Zn = np.conj(Z[(-k) % D])
        return (tw * (Z + Zn) / 2).real * c, (tw * (Z - Zn) / 2j).real * c

    def idct2(a, b):
        def spec(X):
            Xn = np.where(k == 0, 0.0, X[(-k) % D] / c[(-k) % D])
            return np.conj(tw) * (X / c - 1j * Xn) / D
        v = np.fft.ifft(spec(a) + 1j * spec(b)) * D
        xa, xb = np.empty(D), np.empty(D)
        xa[sig], xb[sig] = v.real, v.imag
        return xa, xb

    def pairs(f, M):
        out = np.empty_like(M)
        for j in range(0, M.shape[1], 2):
            b = M[:, j + 1] if j + 1 < M.shape[1] else np.zeros(D)
            ra, rb = f(M[:, j], b)
            out[:, j] = ra
            if j + 1 < M.shape[1]:
                out[:, j + 1] = rb
        return out

    return (lambda M: pairs(dct2, M)), (lambda M: pairs(idct2, M))


def test_dct1_rounding_sensitivity_is_a_reference_property():
    """The reference recursion on its undersampled-DCT workload
    (test_cofem.py:257-265, CG tolerance 1e-4) with the dictionary applied by
    the packed-FFT algorithm of the device's O(D log D) path (exact to 1e-15
    against scipy) takes a different CG step count in one of the 30 E-steps and
    lands alpha ~3e-5 away: the basis of the fast path's alpha tolerance in
    test_gpu_parity::test_reference_dct1d_workload_fast_path."""
    from scipy.fft import dct, idct

    from conftest import golden

    g = golden("reference_workloads.npz")
    D = 1024
    mask = np.sort(g["dct_mask"])
    fdct, fidct = _dct1_packed(D)
    V = np.random.default_rng(0).standard_normal((D, 3))
    assert np.abs(fdct(V) - dct(V, axis=0, norm="ortho")).max() <= 1e-14
    assert np.abs(fidct(V) - idct(V, axis=0, norm="ortho")).max() <= 1e-14
    base = O.dct_op(D, mask)

    def adj(U):
        full = np.zeros((D, U.shape[1]))
        full[mask] = U
        return fdct(full)

    op = O.Op(base.n_rows, D, lambda M: fidct(M)[mask], adj, base.col_sq_norms, base.materialize, "dct")
    cfg = O.CofemConfig(iterations=30, probes=20, seed=0)
    alpha, mu, _, diag = O.run_cofem(op, g["dct_y"], float(g["dct_beta"]), cfg)
    steps = np.array([d["cg_steps"] for d in diag])
    ea = np.linalg.norm(alpha - g["dct_alpha"]) / np.linalg.norm(g["dct_alpha"])
    assert np.any(steps != g["dct_steps"]) and np.abs(steps - g["dct_steps"]).max() <= 2
    assert 1e-5 < ea < 3e-4, ea


def test_ozaki_model_is_close_to_exact():
    rng = np.random.default_rng(3)
    phi = rng.standard_normal((40, 70)).astype(np.float32).astype(np.float64)
    op = O.ozaki_op(phi)
    V = rng.standard_normal((70, 5))
    U = rng.standard_normal((40, 5))
    assert np.abs(op.apply(V) - phi @ V).max() <= 1e-8 * np.abs(phi @ V).max()
    assert np.abs(op.adjoint(U) - phi.T @ U).max() <= 1e-8 * np.abs(phi.T @ U).max()


def _digits4(v):
    """Balanced base-256 digits (ozaki.cuh digits4): v = sum_a d_a 256^(3-a), d_a in [-128, 127]."""
    d = np.zeros((4,) + v.shape, np.int64)
    v = v.copy()
    for a in range(3, -1, -1):
        lo = ((v & 0xFF) ^ 0x80) - 0x80
        d[a] = lo
        v = (v - lo) >> 8
    return d


def test_quantiser_byte_digits_equal_balanced_digits():
    """k_quantize packs the digits as the bytes of (v + 0x80808080) ^ 0x80808080
    (ozaki.cuh); for every |v| <= 2^30 (the fixed-point range) these are the
    balanced digits, and they reconstruct v exactly."""
    rng = np.random.default_rng(0)
    v = np.concatenate([rng.integers(-2**30, 2**30 + 1, 100000),
                        [2**30, -2**30, 0, -1, 1, 127, 128, -128, -129, 255, 256, -256, 2**24, -2**24]]).astype(np.int64)
    d = _digits4(v)
    u = ((v.astype(np.uint64) + 0x80808080) & 0xFFFFFFFF) ^ 0x80808080
    for a in range(4):
        byte = (u >> np.uint64(8 * (3 - a))) & np.uint64(0xFF)
        np.testing.assert_array_equal(((byte ^ np.uint64(0x80)).astype(np.int64) - 0x80), d[a])
    recon = sum(d[a] * (256 ** (3 - a)) for a in range(4))
    np.testing.assert_array_equal(recon, v)
    assert d.min() >= -128 and d.max() <= 127


def test_build_dense_gaussian_matches_reference_draw():
    """operators.py:227-232 draws rng.normal(0, 1/sqrt(N)) in float64: the same
    seed gives the same dictionary and leaves the generator in the same state."""
    from paper_2105_10439_b200 import build_dense_gaussian

    r1, r2 = np.random.default_rng(3), np.random.default_rng(3)
    op = build_dense_gaussian(8, 20, r1)
    np.testing.assert_array_equal(op.matrix, r2.normal(0.0, 1.0 / np.sqrt(8), size=(8, 20)))
    assert op.matrix.dtype == np.float64 and op.kind == "dense-gaussian"
    assert r1.integers(0, 2**32) == r2.integers(0, 2**32)
    f32 = build_dense_gaussian(8, 20, np.random.default_rng(3), dtype=np.float32)
    assert f32.matrix.dtype == np.float32


def test_auto_precision_policy():
    """CgConfig's default precision "auto" resolves per operator."""
    from paper_2105_10439_b200 import CgConfig, ConvolutionOperator, DenseOperator, PartialDct2Operator

    assert CgConfig().precision == "auto"
    with pytest.raises(ValueError):
        CgConfig(precision="fp16")
    assert DenseOperator(np.zeros((256, 1024), dtype=np.float32)).resolve_precision("auto") == "fp64"
    assert DenseOperator(np.zeros((4096, 4097), dtype=np.float32)).resolve_precision("auto") == "ozaki24"
    assert DenseOperator(np.zeros((4, 4), dtype=np.float32)).resolve_precision("ozaki") == "ozaki"
    assert ConvolutionOperator(512, 0.04).resolve_precision("auto") == "fp64"
    h = np.exp(-np.arange(256) / 20.0)
    assert ConvolutionOperator.from_taps(2**22, h).resolve_precision("auto") == "ozaki24"
    assert PartialDct2Operator(64, np.arange(100)).resolve_precision("auto") == "fp64"


def test_float64_workload_alpha_is_summation_order_sensitive():
    """The reference's float64 dense workload (conftest generator, default CG
    tolerance 1e-4, 30 EM iterations): the reference recursion (oracle,
    bit-exact with it) with only the ORDER of the matmul sums permuted moves
    alpha by > 1e-4 -- so no implementation with a different reduction order
    can hold alpha to 1e-4 there (the basis of the 5e-4 alpha bar of
    test_gpu_parity.py::test_reference_dense_float64_parity)."""
    from conftest import golden

    g = golden("reference_workloads.npz")
    phi = g["d64_phi"]
    cfg = O.CofemConfig(iterations=30, probes=20, seed=0)
    base = O.dense_op(phi)
    a0, mu0, _, _ = O.run_cofem(base, g["d64_y"], 1e4, cfg)
    np.testing.assert_array_equal(a0, g["d64_alpha"])
    pc = np.random.default_rng(0).permutation(phi.shape[1])
    pr = np.random.default_rng(1).permutation(phi.shape[0])
    reordered = O.Op(phi.shape[0], phi.shape[1], lambda V: phi[:, pc] @ V[pc], lambda U: phi[pr].T @ U[pr],
                     base.col_sq_norms, base.materialize, "dense")
    a1, mu1, _, _ = O.run_cofem(reordered, g["d64_y"], 1e4, cfg)
    rel_a = np.linalg.norm(a1 - a0) / np.linalg.norm(a0)
    assert 1e-4 < rel_a < 5e-4
    assert np.linalg.norm(mu1 - mu0) / np.linalg.norm(mu0) < 1e-4


def test_dct_pair_step_algebra_against_scipy():
    """The pair-once Makhoul steps the DCT passes implement (csrc/dct.cuh
    pair_op: c_k cancels in the masked pair, one twiddle scaled 1/sqrt(2n)
    serves DCT-II post, DCT-III pre and the fused mask step), emulated in
    numpy in the warp-per-FFT lane / slot distribution, equal scipy's
    orthonormal DCT-II / DCT-III and DCT-III(mask * DCT-II)."""
    import importlib.util
    import os

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "dctw_emul.py")
    spec = importlib.util.spec_from_file_location("dctw_emul", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    for seed in (0, 1):
        for name, err in mod.check(seed).items():
            assert err <= 1e-12, (name, err)


def test_psifree_step_identities_on_a_partial_dct_system():
    """The two identities behind the Psi-free 2-D DCT step (csrc/pcg.cuh
    k_update_psi), checked in numpy along a Jacobi-preconditioned CG run on
    a partial 2-D DCT system: with orthonormal rows pi = <P, A P> equals
    beta ||Phi^T Phi P||^2 + <P, alpha P>, and <P, alpha P> follows the
    direction recurrence P' = eta P + W as eta^2 pap + 2 eta <P, alpha W> +
    <W, alpha W>."""
    from scipy.fft import dctn, idctn

    rng = np.random.default_rng(5)
    n, Q, beta = 32, 5, 1e4
    mask = rng.random((n, n)) < 0.3
    alpha = rng.random(n * n) + 0.5
    gram = lambda X: idctn(mask[..., None] * dctn(X.reshape(n, n, Q), axes=(0, 1), norm="ortho"), axes=(0, 1),
                           norm="ortho").reshape(n * n, Q)  # noqa: E731  Phi^T Phi X
    minv = 1.0 / (beta * 0.3 + alpha)
    B = rng.standard_normal((n * n, Q))
    X, R = np.zeros_like(B), B.copy()
    W = minv[:, None] * R
    P, rho = W.copy(), (R * W).sum(0)
    pap = (W * (alpha[:, None] * W)).sum(0)
    for _ in range(12):
        Z = gram(P)
        pi_direct = (P * (beta * Z + alpha[:, None] * P)).sum(0)
        pi_psifree = beta * (Z * Z).sum(0) + pap
        np.testing.assert_allclose(pi_psifree, pi_direct, rtol=1e-12)
        np.testing.assert_allclose(pap, (P * (alpha[:, None] * P)).sum(0), rtol=1e-12)
        gamma = rho / pi_psifree
        X += gamma * P
        R -= gamma * (beta * Z + alpha[:, None] * P)
        W = minv[:, None] * R
        rho_new = (R * W).sum(0)
        eta = rho_new / rho
        s1, s2 = (P * (alpha[:, None] * W)).sum(0), (W * (alpha[:, None] * W)).sum(0)
        pap = eta * eta * pap + 2.0 * eta * s1 + s2
        P, rho = eta * P + W, rho_new
    assert np.linalg.norm(R) <= 1e-2 * np.linalg.norm(B)  # and it is a converging CG run
