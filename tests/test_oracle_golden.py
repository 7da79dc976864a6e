"""The numpy oracle against golden vectors produced by the real reference.

tests/golden/make_golden.py ran /root/reference/pkg/src/sbl on these seeded
inputs; the oracle (oracle/cofem_oracle.py) must reproduce them.  It does so
bit for bit, because it restates the reference's arithmetic in the same
order -- that is what lets it stand in for the reference on the GPU box.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import cofem_oracle as O
from paper_2105_10439_b200 import simulate as S

PCG = golden("pcg_cases.npz")
VARIANTS = golden("cofem_variants.npz")


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / nb if nb else np.linalg.norm(a)


@pytest.mark.parametrize("name", [str(n) for n in PCG["names"]])
def test_oracle_pcg_matches_reference(name):
    p = lambda k: PCG[f"{name}__{k}"]  # noqa: E731
    beta, tol, steps, printed = p("params")
    op = O.dense_op(p("phi"))
    rep = O.pcg_solve(lambda V: O.system_apply(op, beta, p("alpha"), V), p("B"), p("minv"),
                      O.CgConfig(max_steps=int(steps), tolerance=tol, printed_recursion=bool(printed)))
    assert rep.steps_taken == int(p("steps"))
    np.testing.assert_array_equal(rep.solution, p("X"))
    assert rep.final_relative_residual == float(p("delta"))
    assert rep.converged == bool(p("converged"))
    np.testing.assert_array_equal(rep.breakdown_columns, p("breakdown"))


@pytest.mark.parametrize("name", [str(n) for n in VARIANTS["names"]])
def test_oracle_cofem_variants_match_reference(name):
    p = lambda k: VARIANTS[f"{name}__{k}"]  # noqa: E731
    beta, T, K, U, tol, seed = p("params")
    cfg = O.CofemConfig(iterations=int(T), probes=int(K), seed=int(seed), variant=str(p("variant")),
                        cg=O.CgConfig(max_steps=int(U), tolerance=tol, theta_policy=str(p("policy"))))
    alpha, mu, s, diag = O.run_cofem(O.dense_op(p("phi")), p("y"), beta, cfg)
    np.testing.assert_array_equal(alpha, p("alpha"))
    np.testing.assert_array_equal(mu, p("mu"))
    np.testing.assert_array_equal(s, p("s"))
    assert [d["cg_steps"] for d in diag] == list(p("cg_steps"))


def _config_problem(g, name):
    c = S.CONFIGS[name]
    phi = S.gaussian_dictionary(c.N, c.D, c.seed)
    import hashlib

    assert hashlib.sha256(phi.tobytes()).hexdigest()[:16] == str(g["phi_digest"]), "generator drifted"
    return c, phi


def test_oracle_dense_small_matches_reference():
    g = golden("cofem_dense-small.npz")
    c, phi = _config_problem(g, "dense-small")
    prob, z, _ = S.dense_cs_problem(c, phi=phi)
    np.testing.assert_array_equal(np.asarray(prob.y), g["y"])
    np.testing.assert_array_equal(z, g["z"])
    cfg = O.CofemConfig(iterations=c.T, probes=c.K, seed=c.seed, cg=O.CgConfig(max_steps=c.U, tolerance=c.tol))
    alpha, mu, s, diag = O.run_cofem(O.dense_op(phi), g["y"], c.beta, cfg)
    np.testing.assert_array_equal(alpha, g["alpha"])
    np.testing.assert_array_equal(mu, g["mu"])
    np.testing.assert_array_equal(s, g["s"])
    assert [d["cg_steps"] for d in diag] == list(g["cg_steps"])
    np.testing.assert_array_equal([d["cg_residual"] for d in diag], g["cg_residuals"])


def test_oracle_dense_mid_matches_reference():
    g = golden("cofem_dense-mid_T3.npz")
    c, phi = _config_problem(g, "dense-mid")
    T = int(g["config"][3])
    cfg = O.CofemConfig(iterations=T, probes=c.K, seed=c.seed, cg=O.CgConfig(max_steps=c.U, tolerance=c.tol))
    alpha, mu, s, diag = O.run_cofem(O.dense_op(phi), g["y"], c.beta, cfg)
    np.testing.assert_array_equal(alpha, g["alpha"])
    np.testing.assert_array_equal(mu, g["mu"])
    assert [d["cg_steps"] for d in diag] == list(g["cg_steps"])


def test_oracle_known_answers():
    ka = golden("known_answers.npz")
    # test_cofem.py:187-190 frozen value 2.203363889720147 at mu = s = 1
    v = O.m_step_nonneg(np.array([1.0]), np.array([1.0]))
    assert 1.0 / v[0] == pytest.approx(float(ka["rectified_mu1_s1"][0]), abs=1e-12)
    assert float(ka["rectified_mu1_s1"][0]) == pytest.approx(2.203363889720147, abs=1e-12)
    # test_operators.py:392-394: conv D=3, rho=0.5 -> [1.3125, 1.25, 1]
    conv = O.conv_op(3, 0.5 ** np.arange(3))
    np.testing.assert_allclose(conv.col_sq_norms(), ka["conv3_colsq"], rtol=0, atol=1e-14)
    # test_cg.py:450-453: all-ones, beta 1e4, alpha 1 -> m = 10001
    m = O.make_preconditioner("all-ones", O.dense_op(np.zeros((4, 5))), 1e4, np.ones(5))
    np.testing.assert_array_equal(m, ka["all_ones_m"])


def test_oracle_divergence_and_entry_cases():
    op = O.dense_op(np.eye(4))
    fn = lambda V: O.system_apply(op, 1.0, np.ones(4), V)  # noqa: E731
    with pytest.raises(O.DivergenceError, match="CG step 1"):
        O.pcg_solve(fn, np.full((4, 1), np.inf), np.ones(4), O.CgConfig(max_steps=4, tolerance=1e-12))
    rep = O.pcg_solve(fn, np.zeros((4, 2)), np.ones(4), O.CgConfig(max_steps=5, tolerance=1e-12))
    assert rep.steps_taken == 0 and rep.converged and rep.final_relative_residual == 0.0
    rep = O.pcg_solve(fn, np.ones((4, 1)), np.ones(4), O.CgConfig(max_steps=5, tolerance=1.5))
    assert rep.steps_taken == 0 and rep.final_relative_residual == 1.0


def test_oracle_convolution_matches_reference():
    """oracle conv_op (FFT path) and the run_cofem loop on the reference's own
    convolution workload (simulate.build_problem, dictionary='convolution')."""
    g = golden("conv_cases.npz")
    op = O.conv_op(512, (1.0 - 0.04) ** np.arange(512, dtype=np.float64))  # operators.py:196
    np.testing.assert_array_equal(op.apply(g["V"]), g["fwd"])
    np.testing.assert_array_equal(op.adjoint(g["U"]), g["adj"])
    np.testing.assert_allclose(op.col_sq_norms(), g["colsq"], rtol=1e-14)
    cfg = O.CofemConfig(iterations=20, probes=20, seed=0, cg=O.CgConfig(max_steps=400, tolerance=1e-6))
    alpha, mu, s, diag = O.run_cofem(op, g["y"], float(g["beta"]), cfg)
    assert [d["cg_steps"] for d in diag] == list(g["cg_steps"])
    np.testing.assert_array_equal(mu, g["mu"])
    np.testing.assert_array_equal(alpha, g["alpha"])


def test_convolution_operator_host_side_matches_reference():
    from paper_2105_10439_b200 import ConvolutionOperator, build_exp_convolution

    g = golden("conv_cases.npz")
    op = build_exp_convolution(512, 0.04)
    np.testing.assert_allclose(op.column_sq_norms(), g["colsq"], rtol=1e-14)
    small = ConvolutionOperator(3, 0.5)
    np.testing.assert_allclose(small.column_sq_norms(), [1.3125, 1.25, 1.0], rtol=0, atol=1e-14)
    np.testing.assert_allclose(small.materialize(), [[1, 0, 0], [0.5, 1, 0], [0.25, 0.5, 1]])
    np.testing.assert_allclose(build_exp_convolution(4, 0.04).filter, [1.0, 0.96, 0.9216, 0.884736], atol=1e-15)
    fir = ConvolutionOperator.from_taps(10, [1.0, -0.5, 0.25])
    np.testing.assert_allclose(fir.column_sq_norms()[-2:], [1.25, 1.0])
    with pytest.raises(ValueError):
        ConvolutionOperator(8, 0.0)
    with pytest.raises(ValueError):
        ConvolutionOperator(8, 1.0)
    with pytest.raises(ValueError):
        ConvolutionOperator.from_taps(2, [1.0, 2.0, 3.0])


def test_oracle_reference_workloads():
    """The reference's undersampled-DCT recovery (test_cofem.py:257-265) and a
    float64 dense instance (its conftest generator), bit for bit."""
    g = golden("reference_workloads.npz")
    cfg = O.CofemConfig(iterations=30, probes=20, seed=0)
    alpha, mu, s, diag = O.run_cofem(O.dct_op(1024, g["dct_mask"]), g["dct_y"], float(g["dct_beta"]), cfg)
    np.testing.assert_array_equal(mu, g["dct_mu"])
    np.testing.assert_array_equal(alpha, g["dct_alpha"])
    assert [d["cg_steps"] for d in diag] == list(g["dct_steps"])
    alpha, mu, s, diag = O.run_cofem(O.dense_op(g["d64_phi"]), g["d64_y"], 1e4, cfg)
    np.testing.assert_array_equal(mu, g["d64_mu"])
    np.testing.assert_array_equal(alpha, g["d64_alpha"])


def test_oracle_multitask_matches_reference():
    """run_cofem_multitask (cofem.py:160-214): the shared-support DCT tasks of
    test_cofem.py:295-320 and three dense tasks with shared probes."""
    g = golden("multitask.npz")
    ops = [O.dct_op(256, g[f"dct_mask{l}"]) for l in range(3)]
    cfg = O.CofemConfig(iterations=30, probes=20, seed=42)
    alpha, ests, diag = O.run_cofem_multitask(ops, [g[f"dct_y{l}"] for l in range(3)], 1e4, cfg)
    np.testing.assert_array_equal(alpha, g["dct_alpha"])
    for l, (mu, s) in enumerate(ests):
        np.testing.assert_array_equal(mu, g[f"dct_mu{l}"])
        np.testing.assert_array_equal(s, g[f"dct_s{l}"])
    assert [d["cg_steps"] for d in diag] == list(g["dct_steps"])
    ops = [O.dense_op(g[f"dense_phi{l}"].astype(np.float64)) for l in range(3)]
    cfg = O.CofemConfig(iterations=6, probes=12, seed=3, cg=O.CgConfig(max_steps=400, tolerance=1e-5))
    alpha, ests, diag = O.run_cofem_multitask(ops, [g[f"dense_y{l}"] for l in range(3)], 1e4, cfg,
                                              share_probes=True)
    np.testing.assert_array_equal(alpha, g["dense_alpha"])
    for l, (mu, s) in enumerate(ests):
        np.testing.assert_array_equal(mu, g[f"dense_mu{l}"])
    assert [d["cg_steps"] for d in diag] == list(g["dense_steps"])
