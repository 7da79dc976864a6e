import sys, numpy as np
sys.path.insert(0, '.')
from oracle import cofem_oracle as O
g = np.load('tests/golden/cofem_dense-small.npz')
N, D, K, T, U, tol, beta, seed, frac, sigma = g['config']
from paper_2105_10439_b200 import simulate as S
c = S.CONFIGS['dense-small']
phi = S.gaussian_dictionary(c.N, c.D, c.seed)
op = O.dense_op(phi)
cfg = O.CofemConfig(iterations=int(T), probes=int(K), cg=O.CgConfig(max_steps=int(U), tolerance=tol), seed=int(seed))
a, mu, s, d = O.run_cofem(op, g['y'], beta, cfg)
rel = lambda x, y: np.linalg.norm(x-y)/np.linalg.norm(y)
print('alpha', rel(a, g['alpha']), 'mu', rel(mu, g['mu']), 's', rel(s, g['s']), np.array_equal(a, g['alpha']))
print([x['cg_steps'] for x in d] == list(g['cg_steps']))
pc = np.load('tests/golden/pcg_cases.npz')
for name in pc['names']:
    p = lambda k: pc[f'{name}__{k}']
    beta, tol, steps, printed = p('params')
    opx = O.dense_op(p('phi'))
    fn = lambda V: O.system_apply(opx, beta, p('alpha'), V)
    rep = O.pcg_solve(fn, p('B'), p('minv'), O.CgConfig(max_steps=int(steps), tolerance=tol, printed_recursion=bool(printed)))
    print(name, rep.steps_taken, int(p('steps')), rel(rep.solution, p('X')) if np.linalg.norm(p('X')) else np.abs(rep.solution).max(), rep.final_relative_residual, float(p('delta')), list(rep.breakdown_columns), list(p('breakdown')))
