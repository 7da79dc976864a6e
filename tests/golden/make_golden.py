"""Generate golden vectors by running the REAL reference (build container only).

    SBL_BACKEND=numpy python tests/golden/make_golden.py

Imports the reference package from /root/reference/pkg/src (read-only; it
does not exist on the GPU box) and records its outputs on seeded inputs as
small .npz fixtures next to this script.  The tests check both the numpy
oracle (oracle/) and the CUDA path against these files.  Dictionaries are
drawn float32 so the float32 copy in HBM holds exactly the entries the
float64 reference multiplies.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)
os.environ.setdefault("SBL_BACKEND", "numpy")

import sbl  # noqa: E402  (the reference)
from sbl import cg as ref_cg  # noqa: E402
from sbl import cofem as ref_cofem  # noqa: E402
from sbl.operators import DenseOperator, SystemMatrix  # noqa: E402
from sbl.problem import SblProblem  # noqa: E402

from paper_2105_10439_b200 import simulate as S  # noqa: E402  (problem generator only)


def phi32(rng, n, d):
    return (rng.standard_normal((n, d), dtype=np.float32) * np.float32(1.0 / np.sqrt(n))).astype(np.float32)


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


# ---------------------------------------------------------------- PCG cases --
PCG_CASES = [
    # name, N, D, Q, beta, alpha kind, policy, tol, max_steps, printed, zero_col
    ("exact64", 32, 64, 5, 1e4, "ones", "all-ones", 1e-12, 64, False, None),
    ("capped_jacobi", 16, 48, 3, 1e4, "spread", "jacobi", 1e-5, 10, False, None),
    ("breakdown", 20, 40, 3, 1e4, "spread", "all-ones", 1e-10, 200, False, 1),
    ("printed", 24, 24, 3, 1e2, "spread", "none", 1e-12, 24, True, None),
    ("none_policy", 16, 32, 2, 1e4, "spread", "none", 1e-12, 5, False, None),
    ("wide40", 50, 100, 40, 1e3, "spread", "all-ones", 1e-8, 300, False, None),
    ("odd_dims", 37, 203, 7, 1e4, "spread", "all-ones", 1e-6, 200, False, None),
    ("loose_tol", 32, 64, 4, 1e4, "ones", "all-ones", 0.5, 100, False, None),
]


def make_pcg():
    out = {}
    for i, (name, n, d, q, beta, akind, policy, tol, steps, printed, zc) in enumerate(PCG_CASES):
        rng = np.random.default_rng(1000 + i)
        phi = phi32(rng, n, d)
        alpha = np.ones(d) if akind == "ones" else rng.random(d) + 0.5
        B = rng.standard_normal((d, q))
        if zc is not None:
            B[:, zc] = 0.0
        op = DenseOperator(phi.astype(np.float64))
        sysm = SystemMatrix(op, beta, alpha)
        pre = ref_cg.make_preconditioner(policy, op, beta, alpha)
        rep = ref_cg.solve(sysm, B, pre, ref_cg.CgConfig(max_steps=steps, tolerance=tol, printed_recursion=printed))
        p = f"{name}__"
        out[p + "phi"] = phi
        out[p + "alpha"] = alpha
        out[p + "B"] = B
        out[p + "minv"] = 1.0 / pre.m
        out[p + "params"] = np.array([beta, tol, steps, 1.0 if printed else 0.0])
        out[p + "X"] = rep.solution
        out[p + "steps"] = np.array(rep.steps_taken)
        out[p + "delta"] = np.array(rep.final_relative_residual)
        out[p + "converged"] = np.array(rep.converged)
        out[p + "breakdown"] = rep.breakdown_columns
        print(f"pcg {name}: steps={rep.steps_taken} delta={rep.final_relative_residual:.3e}")
    np.savez_compressed(os.path.join(HERE, "pcg_cases.npz"), names=np.array([c[0] for c in PCG_CASES]), **out)


# ---------------------------------------------------------------- CoFEM -----
def run_reference_cofem(phi, y, beta, cfg):
    problem = SblProblem(y, DenseOperator(phi.astype(np.float64)), beta)
    state, est, diag = ref_cofem.run_cofem(problem, cfg)
    return state, est, diag


def make_cofem_config(cfg_name, iterations=None, fname=None):
    c = S.CONFIGS[cfg_name]
    T = iterations or c.T
    prob, z, phi = S.dense_cs_problem(c)
    rcfg = sbl.CofemConfig(iterations=T, probes=c.K, cg=sbl.CgConfig(max_steps=c.U, tolerance=c.tol), seed=c.seed)
    state, est, diag = run_reference_cofem(phi, np.asarray(prob.y), c.beta, rcfg)
    np.savez_compressed(
        os.path.join(HERE, fname or f"cofem_{cfg_name}.npz"),
        config=np.array([c.N, c.D, c.K, T, c.U, c.tol, c.beta, c.seed, c.frac, c.sigma]),
        phi_digest=np.array(digest(phi)),
        y=np.asarray(prob.y),
        z=z,
        alpha=state.alpha,
        mu=est.mu,
        s=est.s,
        cg_steps=np.array([r["cg_steps"] for r in diag]),
        cg_residuals=np.array([r["cg_residual"] for r in diag]),
    )
    print(f"cofem {cfg_name} T={T}: steps {[r['cg_steps'] for r in diag]}")


VARIANT_CASES = [
    # name, N, D, spikes, T, K, U, tol, variant, policy, seed, beta
    ("nonneg", 64, 128, 6, 10, 8, 200, 1e-6, "nonneg", "all-ones", 5, 1e4),
    ("jacobi", 64, 128, 8, 8, 10, 200, 1e-6, "standard", "jacobi", 6, 1e4),
    # unpreconditioned: a mild beta keeps kappa small enough to converge
    ("none", 48, 96, 5, 2, 6, 400, 1e-8, "standard", "none", 7, 1e1),
    ("single_iteration", 32, 64, 4, 1, 8, 64, 1e-10, "standard", "all-ones", 8, 1e4),
    ("wide_probes", 40, 160, 8, 5, 40, 150, 1e-6, "standard", "all-ones", 9, 1e4),
]


def make_variants():
    out = {}
    for name, n, d, k_sp, T, K, U, tol, variant, policy, seed, beta in VARIANT_CASES:
        rng = np.random.default_rng(seed)
        phi = phi32(rng, n, d)
        z = np.zeros(d)
        sup = rng.choice(d, size=k_sp, replace=False)
        z[sup] = rng.exponential(1.0, size=k_sp) if variant == "nonneg" else rng.standard_normal(k_sp)
        y = phi.astype(np.float64) @ z + 0.01 * rng.standard_normal(n)
        cfg = sbl.CofemConfig(iterations=T, probes=K, seed=seed, variant=variant,
                              cg=sbl.CgConfig(max_steps=U, tolerance=tol, theta_policy=policy))
        state, est, diag = run_reference_cofem(phi, y, beta, cfg)
        p = f"{name}__"
        out[p + "phi"] = phi
        out[p + "y"] = y
        out[p + "params"] = np.array([beta, T, K, U, tol, seed])
        out[p + "variant"] = np.array(variant)
        out[p + "policy"] = np.array(policy)
        out[p + "alpha"] = state.alpha
        out[p + "mu"] = est.mu
        out[p + "s"] = est.s
        out[p + "cg_steps"] = np.array([r["cg_steps"] for r in diag])
        out[p + "cg_residuals"] = np.array([r["cg_residual"] for r in diag])
        print(f"variant {name}: steps {[r['cg_steps'] for r in diag]}")
    np.savez_compressed(os.path.join(HERE, "cofem_variants.npz"), names=np.array([c[0] for c in VARIANT_CASES]),
                        **out)


def make_conv():
    """Reference ConvolutionOperator (operators.py:182-225): apply / adjoint /
    column norms, and run_cofem on the reference's own convolution workload
    (simulate.build_problem with dictionary='convolution')."""
    from sbl.operators import ConvolutionOperator
    from sbl.simulate import ExperimentSpec, build_problem

    rng = np.random.default_rng(77)
    op = ConvolutionOperator(512, 0.04)
    V = rng.standard_normal((512, 21))
    U = rng.standard_normal((512, 5))
    out = {"V": V, "U": U, "fwd": op.apply(V), "adj": op.apply_adjoint(U), "colsq": op.column_sq_norms()}
    spec = ExperimentSpec(dictionary="convolution", D=512, rho=0.04, seed=400,  # data seed; cofem seed 0
                          cofem=sbl.CofemConfig(iterations=20, probes=20,
                                                cg=sbl.CgConfig(max_steps=400, tolerance=1e-6)))
    problem, z = build_problem(spec)
    state, est, diag = ref_cofem.run_cofem(problem, spec.cofem)
    out.update(y=np.asarray(problem.y), z=z, beta=np.array(problem.beta), alpha=state.alpha, mu=est.mu,
               s=est.s, cg_steps=np.array([r["cg_steps"] for r in diag]))
    print(f"conv cofem steps {[r['cg_steps'] for r in diag]}")
    np.savez_compressed(os.path.join(HERE, "conv_cases.npz"), **out)


def make_reference_workloads():
    """Two workloads the reference's own tests use: the undersampled-DCT
    recovery of test_cofem.py:257-265 and a float64 dense instance from its
    conftest generator (tests/conftest.py:10-24)."""
    from sbl.operators import build_undersampled_dct
    from sbl.problem import substream
    from sbl.simulate import gen_observation, gen_signal

    op = build_undersampled_dct(1024, 341, substream(0, 0))
    z = gen_signal(1024, 122, "normal", substream(0, 1))
    y, beta = gen_observation(op, z, 0.01, substream(0, 2))
    cfg = sbl.CofemConfig(iterations=30, probes=20, seed=0)
    state, est, diag = ref_cofem.run_cofem(SblProblem(y, op, beta), cfg)
    out = {"dct_mask": op.mask, "dct_y": y, "dct_z": z, "dct_beta": np.array(beta), "dct_mu": est.mu,
           "dct_alpha": state.alpha, "dct_steps": np.array([r["cg_steps"] for r in diag])}
    print(f"dct1d steps {[r['cg_steps'] for r in diag]}")
    rng = np.random.default_rng(12345)
    n_rows, dim, n_spikes, beta = 64, 256, 15, 1e4
    phi = rng.normal(0.0, 1.0 / np.sqrt(n_rows), size=(n_rows, dim))
    zz = np.zeros(dim)
    zz[rng.choice(dim, size=n_spikes, replace=False)] = rng.uniform(-2.0, 2.0, size=n_spikes)
    yy = phi @ zz + (1.0 / np.sqrt(beta)) * rng.standard_normal(n_rows)
    cfg = sbl.CofemConfig(iterations=30, probes=20, seed=0)
    state, est, diag = ref_cofem.run_cofem(SblProblem(yy, DenseOperator(phi), beta), cfg)
    out.update(d64_phi=phi, d64_y=yy, d64_z=zz, d64_mu=est.mu, d64_alpha=state.alpha,
               d64_steps=np.array([r["cg_steps"] for r in diag]))
    print(f"dense64 steps {[r['cg_steps'] for r in diag]}")
    np.savez_compressed(os.path.join(HERE, "reference_workloads.npz"), **out)


def make_multitask():
    """run_cofem_multitask (cofem.py:160-214) on the reference's shared-support
    undersampled-DCT tasks (test_acceptance.py:367-378 / test_cofem.py:295-320,
    seed 42) and on three float32 dense tasks with shared probes."""
    from sbl.operators import build_undersampled_dct
    from sbl.problem import MultiTaskProblem, substream

    out = {}
    dim, n_rows, n_spikes, L, seed = 256, 85, 16, 3, 42
    support = substream(seed, 1).choice(dim, size=n_spikes, replace=False)
    tasks = []
    for ell in range(L):
        op = build_undersampled_dct(dim, n_rows, substream(seed, 0, ell))
        z = np.zeros(dim)
        z[support] = substream(seed, 1, ell).normal(0.0, np.sqrt(5.0), size=n_spikes)
        y = op.apply(z) + 0.01 * substream(seed, 2, ell).standard_normal(n_rows)
        tasks.append(SblProblem(y, op, 1e4))
        out[f"dct_mask{ell}"] = op.mask
        out[f"dct_y{ell}"] = y
    cfg = sbl.CofemConfig(iterations=30, probes=20, seed=seed)
    state, ests, diag = ref_cofem.run_cofem_multitask(MultiTaskProblem(tuple(tasks)), cfg)
    out["dct_support"] = np.sort(support)
    out["dct_alpha"] = state.alpha
    for ell, e in enumerate(ests):
        out[f"dct_mu{ell}"] = e.mu
        out[f"dct_s{ell}"] = e.s
    out["dct_steps"] = np.array([r["cg_steps"] for r in diag])
    print(f"multitask dct steps {[r['cg_steps'] for r in diag]}")

    rng = np.random.default_rng(77)
    n, d = 96, 384
    tasks = []
    zs = np.zeros(d)
    zs[rng.choice(d, size=12, replace=False)] = 1.0
    for ell in range(L):
        phi = phi32(rng, n, d)
        z = zs * rng.standard_normal(d)
        y = phi.astype(np.float64) @ z + 0.01 * rng.standard_normal(n)
        tasks.append(SblProblem(y, DenseOperator(phi.astype(np.float64)), 1e4))
        out[f"dense_phi{ell}"] = phi
        out[f"dense_y{ell}"] = y
    cfg = sbl.CofemConfig(iterations=6, probes=12, seed=3, cg=sbl.CgConfig(max_steps=400, tolerance=1e-5))
    state, ests, diag = ref_cofem.run_cofem_multitask(MultiTaskProblem(tuple(tasks)), cfg, share_probes=True)
    out["dense_alpha"] = state.alpha
    for ell, e in enumerate(ests):
        out[f"dense_mu{ell}"] = e.mu
        out[f"dense_s{ell}"] = e.s
    out["dense_steps"] = np.array([r["cg_steps"] for r in diag])
    out["dense_resid"] = np.array([r["cg_residual"] for r in diag])
    print(f"multitask dense steps {[r['cg_steps'] for r in diag]}")
    np.savez_compressed(os.path.join(HERE, "multitask.npz"), **out)


def make_known_answers():
    """Known-answer values the reference's own tests pin (test_cofem.py:187-190,
    test_cg.py:450-466, test_operators.py:392-394), recomputed from the reference."""
    from sbl.cofem import _rectified_second_moment
    from sbl.operators import ConvolutionOperator

    out = {
        "rectified_mu1_s1": _rectified_second_moment(np.array([1.0]), np.array([1.0]), 1e-12),
        "conv3_colsq": ConvolutionOperator(3, 0.5).column_sq_norms(),
        "all_ones_m": ref_cg.make_preconditioner("all-ones", DenseOperator(np.zeros((4, 5))), 1e4, np.ones(5)).m,
    }
    np.savez_compressed(os.path.join(HERE, "known_answers.npz"), **out)


if __name__ == "__main__":
    which = set(sys.argv[1:]) or {"known", "pcg", "variants", "small", "mid", "conv", "workloads",
                                    "multitask"}
    if "known" in which:
        make_known_answers()
    if "conv" in which:
        make_conv()
    if "workloads" in which:
        make_reference_workloads()
    if "multitask" in which:
        make_multitask()
    if "pcg" in which:
        make_pcg()
    if "variants" in which:
        make_variants()
    if "small" in which:
        make_cofem_config("dense-small")
    if "mid" in which:
        make_cofem_config("dense-mid", iterations=3, fname="cofem_dense-mid_T3.npz")
