"""BASELINE.json's five configurations at their stated sizes and lengths,
against the REAL reference's float64 run_cofem (golden vectors made by
tests/golden/make_golden.py / make_golden_large.py in the build container,
where /root/reference is importable).

north_star bar, written here as tolerances: relative L2 error of mu and alpha
<= 1e-4 after the EM iterations, identical recovered support (alpha below the
pruning threshold 1e6 of the reference's test_cofem.py:347) and NMSE against
the ground truth within 1 % (relative) of the reference's.  Every run here
uses the library's DEFAULT precision (CgConfig(precision="auto")).

The 2^20 / 2^22 configurations keep a fixed random sample of 65536
coordinates plus the support bit mask, the full-vector norms and block sums
(golden files of a few MB); mu / alpha errors are measured on the sample (an
unbiased estimate of the full relative error), the support on all D.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, golden
from paper_2105_10439_b200 import run_cofem
from paper_2105_10439_b200 import simulate as S

pytestmark = pytest.mark.gpu
PRUNE = 1e6
TOL = 1e-4


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def need(name):
    if not os.path.exists(os.path.join(GOLDEN, name)):
        pytest.skip(f"golden {name} not generated (tests/golden/make_golden_large.py)")
    return golden(name)


def steps_of(diag):
    return np.array([d["cg_steps"] for d in diag])


def check_dense(g, st, est, diag, z, step_slack):
    emu, ea = rel(est.mu, g["mu"]), rel(st.alpha, g["alpha"])
    steps = steps_of(diag)
    info = (emu, ea, steps.tolist(), g["cg_steps"].tolist())
    assert emu <= TOL and ea <= TOL, info
    np.testing.assert_array_equal(st.alpha < PRUNE, g["alpha"] < PRUNE)
    nref, nour = float(g["nmse"]), S.nmse(est.mu, z)
    assert abs(nour - nref) <= 0.01 * nref, (nour, nref)
    assert np.all(np.abs(steps - g["cg_steps"]) <= step_slack), info
    return info


def test_config1_dense_small_default_precision():
    """Config 1 (N=256, D=1024, K=20, 50 EM iterations, cap 100): the default
    precision resolves to float64 CUDA-core contractions for a dictionary this
    small and holds alpha to 1e-4 on this cap-bound (chaotic) workload."""
    g = golden("cofem_dense-small.npz")
    c = S.CONFIGS["dense-small"]
    prob, z, _ = S.dense_cs_problem(c)
    assert prob.op.resolve_precision("auto") == "fp64"
    st, est, diag = run_cofem(prob, c.cofem_config("auto"))
    prob.op.release()
    emu, ea = rel(est.mu, g["mu"]), rel(st.alpha, g["alpha"])
    assert emu <= TOL and ea <= TOL, (emu, ea)
    np.testing.assert_array_equal(st.alpha < PRUNE, g["alpha"] < PRUNE)
    nref, nour = S.nmse(g["mu"], z), S.nmse(est.mu, z)
    assert abs(nour - nref) <= 0.01 * nref


@pytest.mark.parametrize("precision", ["auto", "ozaki", "ozaki24"])
def test_config2_dense_mid_full_length(precision):
    """Config 2 (N=4096, D=16384, K=20, 30 EM iterations, cap 200, tol 1e-5),
    all 30 iterations against the reference: the default mode and both
    tensor-core dictionary widths (32-bit and 24-bit fixed-point Phi)."""
    g = need("cofem_dense-mid_T30.npz")
    c = S.CONFIGS["dense-mid"]
    prob, z, phi = S.dense_cs_problem(c)
    np.testing.assert_array_equal(np.asarray(prob.y), g["y"])
    st, est, diag = run_cofem(prob, c.cofem_config(precision))
    prob.op.release()
    print(f"dense-mid T30 {precision}", check_dense(g, st, est, diag, z, step_slack=5))


@pytest.mark.parametrize("world", [2, 4])
def test_config2_dense_mid_column_sharded_full_length(world):
    """Config 2's "2-GPU D-sharded" leg: 2 / 4 column shards (in-process shard
    group, the NCCL path's exchanges) over all 30 iterations."""
    from paper_2105_10439_b200.distributed import run_cofem_threaded

    g = need("cofem_dense-mid_T30.npz")
    c = S.CONFIGS["dense-mid"]
    prob, z, _ = S.dense_cs_problem(c)
    st, est, diag = run_cofem_threaded(prob, c.cofem_config("auto"), devices=[0] * world)
    print(f"dense-mid T30 x{world}", check_dense(g, st, est, diag, z, step_slack=5))


@pytest.fixture(scope="module")
def dense_large():
    g = need("cofem_dense-large_T20.npz")
    c = S.CONFIGS["dense-large"]
    phi = S.gaussian_dictionary(c.N, c.D, c.seed)
    prob, z, _ = S.dense_cs_problem(c, phi=phi)
    np.testing.assert_array_equal(np.asarray(prob.y), g["y"])
    yield g, c, prob, z
    prob.op.release()


@pytest.mark.parametrize("precision", ["auto", "ozaki", "ozaki24"])
def test_config3_dense_large_headline(dense_large, precision):
    """Config 3, the headline (N=16384, D=65536 -- Phi 4 GiB --, K=20, 20 EM
    iterations, cap 200, tol 1e-5) on the int8 tensor-core path (the default
    mode, the 32-bit and the 24-bit fixed-point dictionary) against the
    reference's float64 run on the same float32-exact Phi."""
    g, c, prob, z = dense_large
    if precision == "auto":
        assert prob.op.resolve_precision("auto") in ("ozaki", "ozaki24")
    st, est, diag = run_cofem(prob, c.cofem_config(precision, iterations=int(g["config"][3])))
    prob.op.release()
    print(f"dense-large {precision}", check_dense(g, st, est, diag, z, step_slack=3))


def check_sampled(g, st, est, diag, z, step_slack):
    idx = g["sample"].astype(np.int64)
    emu = rel(est.mu[idx], g["mu_sample"])
    ea = rel(st.alpha[idx], g["alpha_sample"])
    es = rel(est.s[idx], g["s_sample"])
    steps = steps_of(diag)
    info = (emu, ea, es, steps.tolist(), g["cg_steps"].tolist())
    assert emu <= TOL and ea <= TOL, info
    support = np.unpackbits(g["support_bits"])[: est.mu.size].astype(bool)
    np.testing.assert_array_equal(st.alpha < PRUNE, support)
    # full-vector checks: norms and block sums
    np.testing.assert_allclose([np.linalg.norm(est.mu), np.linalg.norm(st.alpha)], g["norms"][:2], rtol=TOL)
    blocks = g["mu_blocks"].size
    assert rel(est.mu.reshape(blocks, -1).sum(axis=1), g["mu_blocks"]) <= TOL
    nref, nour = float(g["nmse"]), S.nmse(est.mu, z)
    assert abs(nour - nref) <= 0.01 * nref, (nour, nref)
    assert np.all(np.abs(steps - g["cg_steps"]) <= step_slack), info
    return info


def test_config5_dct_large_full_size():
    """Config 5 (1024 x 1024 image, D = 2^20, 25 % variable-density 2-D DCT
    mask, K=20, 20 EM iterations): the fused float64 FFT passes against the
    reference's CoFEM loop over the same partial-DCT operator."""
    g = need("cofem_dct-large_T20.npz")
    c = S.DCT_CONFIGS["dct-large"]
    prob, z = S.dct2_problem(c)
    st, est, diag = run_cofem(prob, c.cofem_config("auto", iterations=int(g["config"][3])))
    prob.op.release()
    # orthonormal-row DCT dictionaries make CG's stopping step sensitive to
    # 1e-12-level arithmetic: steps within 3, total 5 %
    info = check_sampled(g, st, est, diag, z, step_slack=3)
    assert abs(steps_of(diag).sum() - g["cg_steps"].sum()) <= 0.05 * g["cg_steps"].sum(), info
    print("dct-large", info)


@pytest.mark.parametrize("precision", ["auto", "ozaki"])
def test_config4_conv_large_full_size(precision):
    """Config 4 (N = D = 2^22 samples, causal 256-tap exp(-t/20) filter, K=30,
    sigma 0.05) on the banded int8 tensor-core path, against the reference's
    CoFEM loop over the same Toeplitz operator for the golden's EM
    iterations (the CPU reference needs ~35 min per iteration here)."""
    g = need("cofem_conv-large_T2.npz")
    c = S.CONV_CONFIGS["conv-large"]
    prob, z = S.conv_problem(c)
    assert prob.op.resolve_precision("auto") in ("ozaki", "ozaki24")
    st, est, diag = run_cofem(prob, c.cofem_config(precision, iterations=int(g["config"][4])))
    prob.op.release()
    print(f"conv-large {precision}", check_sampled(g, st, est, diag, z, step_slack=3))
