"""Sharded execution on one GPU through the in-process shard group.

The ranks of a sharded problem run as host threads of one process, each on
its own context and stream; the library's exchanges (all-reduce sum / max,
neighbour halo send/recv) run between them through stream-ordered events --
the same code path as the NCCL communicator up to the transport, so the
sharding arithmetic (column shards of a dense Phi, time shards of a
convolution with halo exchange) is checked on the one available GPU.

* convolution apply / adjoint: time shards reproduce the unsharded banded
  contraction BITWISE (the ranks agree on the int8 scales through the max
  all-reduce, and every output row sees the same operand window);
* convolution CoFEM: same CG step counts as the unsharded run, mu / alpha
  equal up to the summation order of the PCG dot products (~5e-9);
* dense CoFEM: column shards (sharing the whole dictionary's row scales and
  the operand scales) against the float64 oracle / the reference's golden
  run, and against the one-GPU run (same CG steps, mu / alpha to 1e-7).
"""

import numpy as np
import pytest

from oracle import cofem_oracle as O
from paper_2105_10439_b200 import ConvolutionOperator, DenseOperator, SblProblem, run_cofem
from paper_2105_10439_b200 import simulate as S
from paper_2105_10439_b200.distributed import (
    run_cofem_threaded,
    run_threaded,
    threaded_contexts,
)

pytestmark = pytest.mark.gpu
PRUNE = 1e6


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def exp_taps(ntaps, tau=20.0):
    h = np.exp(-np.arange(ntaps) / tau)
    return h / np.linalg.norm(h)


def sharded_apply(op, X, world, adjoint=False):
    contexts, shards = threaded_contexts(op, "ozaki", [0] * world)
    try:
        parts = run_threaded(world, lambda r: (contexts[r].apply_adjoint if adjoint else contexts[r].apply)(
            np.ascontiguousarray(X[shards[r][0]:shards[r][1]])), contexts[0].group)
    finally:
        for c in contexts:
            c.close()
    return np.concatenate(parts, axis=0)


@pytest.mark.parametrize("dim,ntaps,world,q", [(4096, 256, 2, 31), (4096, 256, 3, 8), (5000, 100, 4, 21),
                                               (2048, 257, 2, 1), (1536, 64, 5, 40)])
def test_time_sharded_convolution_apply_is_bitwise(dim, ntaps, world, q):
    h = exp_taps(ntaps)
    op = ConvolutionOperator.from_taps(dim, h)
    rng = np.random.default_rng(dim + world)
    V = rng.standard_normal((dim, q))
    ctx = op.context("ozaki")  # the unsharded int8 band path (plain apply may pick the fp64 FFT path)
    full_f, full_a = ctx.apply(V), ctx.apply_adjoint(V)
    np.testing.assert_array_equal(sharded_apply(op, V, world), full_f)
    np.testing.assert_array_equal(sharded_apply(op, V, world, adjoint=True), full_a)
    # and both are the convolution (float64 numpy) to the int8 path's accuracy
    ref = np.stack([np.convolve(V[:, k], h)[:dim] for k in range(q)], axis=1)
    assert rel(full_f, ref) <= 1e-8


@pytest.mark.parametrize("world,K", [(2, 20), (3, 20), (2, 40)])
def test_time_sharded_convolution_cofem_matches_unsharded(world, K):
    """K = 40: two column chunks per contraction, each with its own halo exchange."""
    c = S.ConvConfig("conv-shard", 8192, 256, 20.0, 0.01, 0.05, K, 3, 200, 1e-5)
    prob, z = S.conv_problem(c)
    cfg = c.cofem_config("ozaki")
    st1, est1, d1 = run_cofem(prob, cfg)
    st2, est2, d2 = run_cofem_threaded(prob, cfg, devices=[0] * world)
    assert [d["cg_steps"] for d in d1] == [d["cg_steps"] for d in d2]
    # the shards' dot products sum in another order; the int8 operand rounding
    # turns those last-bit differences into ~1e-9-level ones
    assert rel(est2.mu, est1.mu) <= 1e-7 and rel(st2.alpha, st1.alpha) <= 1e-7
    np.testing.assert_array_equal(st2.alpha < PRUNE, st1.alpha < PRUNE)


@pytest.mark.parametrize("precision,world", [("ozaki", 2), ("ozaki", 3), ("fp64", 2)])
def test_column_sharded_dense_cofem_matches_oracle(precision, world):
    """Dense column shards: the partial Phi_r P_r all-reduce, then each rank
    re-derives the V column maxima (same row scales everywhere, so the same
    V scales) for its Phi_r^T quantisation."""
    rng = np.random.default_rng(5)
    n, d = 512, 2048
    phi = (rng.standard_normal((n, d)) / np.sqrt(n)).astype(np.float32)
    z = np.zeros(d)
    z[rng.choice(d, 40, replace=False)] = rng.standard_normal(40)
    y = phi.astype(np.float64) @ z + 0.01 * rng.standard_normal(n)
    prob = SblProblem(y, DenseOperator(phi), 1e4)
    from paper_2105_10439_b200 import CgConfig, CofemConfig

    cfg = CofemConfig(iterations=4, probes=12, seed=1, cg=CgConfig(max_steps=200, tolerance=1e-5, precision=precision))
    st, est, diag = run_cofem_threaded(prob, cfg, devices=[0] * world)
    ocfg = O.CofemConfig(iterations=4, probes=12, seed=1, cg=O.CgConfig(max_steps=200, tolerance=1e-5))
    alpha, mu, s, odiag = O.run_cofem(O.dense_op(phi), y, 1e4, ocfg)
    assert rel(est.mu, mu) <= 1e-4 and rel(st.alpha, alpha) <= 1e-4
    # ~180-step solves at beta = 1e4: 1e-9-level contraction differences move
    # the stopping step by a step or two (the unsharded int8 path does too)
    assert np.all(np.abs(np.array([x["cg_steps"] for x in diag]) - [x["cg_steps"] for x in odiag]) <= 3)
    np.testing.assert_array_equal(st.alpha < PRUNE, alpha < PRUNE)


def test_group_failure_releases_the_other_ranks():
    """A rank that fails outside an exchange breaks the group: the others
    return an error instead of waiting at the next barrier."""
    op = ConvolutionOperator.from_taps(2048, exp_taps(64))
    contexts, shards = threaded_contexts(op, "ozaki", [0, 0])
    V = np.ones((2048, 3))

    def body(r):
        if r == 1:
            raise RuntimeError("host-side failure before the first exchange")
        return contexts[r].apply(V[shards[r][0]:shards[r][1]])

    try:
        with pytest.raises(RuntimeError, match="host-side failure"):
            run_threaded(2, body, contexts[0].group)
    finally:
        for c in contexts:
            c.close()


@pytest.mark.parametrize("world", [2, 4])
def test_dense_mid_column_sharded_matches_reference_golden(world):
    """BASELINE config 2 (N=4096, D=16384, K=20, 2-GPU D-sharded) as 2 / 4
    column shards against the reference's own float64 run (golden vectors,
    3 EM iterations): mu, alpha within 1e-5 (the bar is 1e-4), same support."""
    from conftest import golden

    g = golden("cofem_dense-mid_T3.npz")
    c = S.CONFIGS["dense-mid"]
    prob, z, _ = S.dense_cs_problem(c)
    T = int(g["config"][3])
    cfg = c.cofem_config("ozaki", iterations=T)
    st, est, diag = run_cofem_threaded(prob, cfg, devices=[0] * world)
    assert rel(est.mu, g["mu"]) <= 1e-5 and rel(st.alpha, g["alpha"]) <= 1e-5
    np.testing.assert_array_equal(st.alpha < PRUNE, g["alpha"] < PRUNE)
    assert np.all(np.abs(np.array([d["cg_steps"] for d in diag]) - g["cg_steps"]) <= 3)
    # the shards share the unsharded row / operand scales: they track the
    # one-GPU run up to the fp64 summation order of the partial products
    st1, est1, diag1 = run_cofem(prob, cfg)
    prob.op.release()
    assert [d["cg_steps"] for d in diag] == [d["cg_steps"] for d in diag1]
    assert rel(est.mu, est1.mu) <= 1e-7 and rel(st.alpha, st1.alpha) <= 1e-7
