import numpy as np, time, sys
sys.path.insert(0, '.')
from oracle import cofem_oracle as O
exec(open('scratch/fp32_study.py').read().split("N, D, T, U =")[0].split("from oracle import cofem_oracle as O")[1])
N, D, T, U = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
phi, z, y = problem(N, D, 0.05 if D<=1024 else 0.02, 0.01, 0)
beta = 1e4
op64 = O.dense_op(phi)
cfg = O.CofemConfig(iterations=T, probes=20, cg=O.CgConfig(max_steps=U, tolerance=1e-5))
rng = O.substream(0, 3)
probes = [O.draw_rademacher(D, 20, rng) for _ in range(T)]
a64, mu64, s64, d64 = O.run_cofem(op64, y, beta, cfg, probes_seq=probes)
phi64 = phi.astype(np.float64)
def run(mode):
    alpha = np.ones(D); diag=[]
    for t in range(T):
        rhs = np.concatenate([probes[t], (phi64.T @ y)[:, None]], axis=1)
        minv = 1.0 / (beta + alpha)
        if mode == 'gemm32acc32':   # vectors f64, operands rounded to f32, f32 accumulate
            fn = lambda V: beta * (phi.T @ (phi @ V.astype(np.float32))).astype(np.float64) + alpha[:, None]*V
        elif mode == 'gemm32acc64': # operands rounded to f32, exact accumulate
            fn = lambda V: beta * (phi64.T @ (phi64 @ V.astype(np.float32).astype(np.float64)).astype(np.float32).astype(np.float64)) + alpha[:, None]*V
        elif mode == 'gemm32acc32_u64':   # forward rounds V to fp32, U kept f32
            fn = lambda V: beta * (phi.T @ (phi @ V.astype(np.float32))).astype(np.float64) + alpha[:, None]*V
        rep = O.pcg_solve(fn, rhs, minv, cfg.cg, dtype=np.float64)
        sol = rep.solution
        mu = beta * sol[:, 20]; s = (probes[t] * sol[:, :20]).mean(axis=1)
        if t < T-1: alpha = O.m_step(mu, s)
        diag.append(rep.steps_taken)
    return alpha, mu, s, diag
rel = lambda a,b: np.linalg.norm(a-b)/np.linalg.norm(b)
for mode in sys.argv[5:]:
    a, mu, s, d = run(mode)
    print(mode, 'steps', d[:3], d[-3:], 'rel mu %.2e alpha %.2e s %.2e' % (rel(mu, mu64), rel(a, a64), rel(s, s64)))
