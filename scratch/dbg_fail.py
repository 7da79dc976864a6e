import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import golden
from oracle import cofem_oracle as O
from paper_2105_10439_b200 import *
from paper_2105_10439_b200 import _lib, simulate as S
rel = lambda a, b: np.linalg.norm(a-b)/np.linalg.norm(b)
PCG = golden('pcg_cases.npz')
for name in PCG['names']:
    p = lambda k: PCG[f'{name}__{k}']
    beta, tol, steps, printed = p('params')
    sysm = SystemMatrix(DenseOperator(p('phi')), beta, p('alpha'))
    for prec in ('fp64', 'ozaki', 'fp32'):
        rep = solve(sysm, p('B'), Preconditioner(m=1.0/p('minv')), CgConfig(max_steps=int(steps), tolerance=tol, printed_recursion=bool(printed), precision=prec))
        print('pcg', name, prec, rep.steps_taken, int(p('steps')), 'conv', rep.converged, bool(p('converged')), 'rel %.2e' % rel(rep.solution, p('X')), 'delta %.3e ref %.3e' % (rep.final_relative_residual, float(p('delta'))))
rng = np.random.default_rng(5)
phi = (rng.standard_normal((20, 60)) / np.sqrt(20)).astype(np.float32)
op = DenseOperator(phi); alpha = rng.random(60) + 0.5; sysm = SystemMatrix(op, 50.0, alpha)
Ba, Bb = rng.standard_normal((60, 3)), rng.standard_normal((60, 2))
pa = make_preconditioner("all-ones", op, 50.0, alpha); pb = Preconditioner(m=50.0 * (rng.random(60) + 0.5) + alpha)
rep, slices = solve_blocked([sysm, sysm], [Ba, Bb], [pa, pb], CgConfig(max_steps=400, tolerance=1e-12, precision="fp64"))
minv = np.concatenate([np.repeat((1.0 / pa.m)[:, None], 3, 1), np.repeat((1.0 / pb.m)[:, None], 2, 1)], 1)
oref = O.pcg_solve(lambda V: O.system_apply(O.dense_op(phi), 50.0, alpha, V), np.concatenate([Ba, Bb], 1), minv, O.CgConfig(max_steps=400, tolerance=1e-12))
print('blocked', rep.steps_taken, oref.steps_taken, rel(rep.solution, oref.solution), rep.final_relative_residual, oref.final_relative_residual)
V = golden('cofem_variants.npz')
for name in V['names']:
    p = lambda k: V[f'{name}__{k}']
    beta, T, K, U, tol, seed = p('params')
    prob = SblProblem(p('y'), DenseOperator(p('phi')), beta)
    for prec in ('fp64', 'ozaki', 'fp32'):
        cfg = CofemConfig(iterations=int(T), probes=int(K), seed=int(seed), variant=str(p('variant')), cg=CgConfig(max_steps=int(U), tolerance=tol, theta_policy=str(p('policy')), precision=prec))
        st, est, diag = run_cofem(prob, cfg)
        print('var', name, prec, 'mu %.2e alpha %.2e s %.2e' % (rel(est.mu, p('mu')), rel(st.alpha, p('alpha')), rel(est.s, p('s'))), [d['cg_steps'] for d in diag], list(p('cg_steps')), 'supp', np.array_equal(st.alpha<1e6, p('alpha')<1e6))
g = golden('cofem_dense-mid_T3.npz'); c = S.CONFIGS['dense-mid']
prob, z, _ = S.dense_cs_problem(c)
for prec in ('fp64', 'ozaki', 'fp32'):
    st, est, diag = run_cofem(prob, c.cofem_config(prec, iterations=3))
    print('mid', prec, 'mu %.2e alpha %.2e' % (rel(est.mu, g['mu']), rel(st.alpha, g['alpha'])), [d['cg_steps'] for d in diag], list(g['cg_steps']), 'supp', np.array_equal(st.alpha<1e6, g['alpha']<1e6))
