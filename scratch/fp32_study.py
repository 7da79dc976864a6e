import numpy as np, time, sys
sys.path.insert(0, '.')
from oracle import cofem_oracle as O

def problem(N, D, frac, sigma, seed):
    phi = (O.substream(seed, 0).standard_normal((N, D), dtype=np.float32) * np.float32(1/np.sqrt(N)))
    rs = O.substream(seed, 1)
    d = int(round(frac * D))
    z = np.zeros(D); z[rs.choice(D, size=d, replace=False)] = rs.standard_normal(d)
    y = phi.astype(np.float64) @ z + sigma * O.substream(seed, 2).standard_normal(N)
    return phi, z, y

N, D, T, U = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
phi, z, y = problem(N, D, 0.05 if D<=1024 else 0.02, 0.01, 0)
beta = 1e4
op64 = O.dense_op(phi)
cfg = O.CofemConfig(iterations=T, probes=20, cg=O.CgConfig(max_steps=U, tolerance=1e-5))
rng = O.substream(0, 3)
probes = [O.draw_rademacher(D, 20, rng) for _ in range(T)]
t=time.time(); a64, mu64, s64, d64 = O.run_cofem(op64, y, beta, cfg, probes_seq=probes); print('fp64', time.time()-t)
# fp32 emulation: float32 matmuls
phi32 = phi
class Op32: pass
op32 = O.Op(N, D, lambda V: phi32 @ V.astype(np.float32), lambda Uu: phi32.T @ Uu.astype(np.float32), op64.col_sq_norms, op64.materialize)
def run32():
    alpha = np.ones(D); diag=[]
    for t in range(T):
        rhs = np.concatenate([probes[t], (phi.T.astype(np.float64) @ y)[:, None]], axis=1)
        minv = 1.0 / (beta + alpha)
        a32 = alpha.astype(np.float32); b32=np.float32(beta)
        fn = lambda V: (b32 * (phi32.T @ (phi32 @ V)) + a32[:, None] * V).astype(np.float32)
        rep = O.pcg_solve(fn, rhs, minv, cfg.cg, dtype=np.float32)
        sol = rep.solution.astype(np.float64)
        mu = beta * sol[:, 20]; s = (probes[t] * sol[:, :20]).mean(axis=1)
        if t < T-1: alpha = O.m_step(mu, s)
        diag.append(rep.steps_taken)
    return alpha, mu, s, diag
t=time.time(); a32, mu32, s32, d32 = run32(); print('fp32', time.time()-t)
rel = lambda a,b: np.linalg.norm(a-b)/np.linalg.norm(b)
print('steps64', [d['cg_steps'] for d in d64]); print('steps32', d32)
print('rel mu', rel(mu32, mu64), 'rel alpha', rel(a32, a64), 'rel s', rel(s32, s64))
la = np.log10(a64); la32=np.log10(a32)
print('max |log10 alpha diff|', np.abs(la-la32).max())
th = 1e6
print('support64', (a64<th).sum(), 'support32', (a32<th).sum(), 'same', np.array_equal(a64<th, a32<th))
nm = lambda m: np.linalg.norm(m-z)**2/np.linalg.norm(z)**2
print('nmse64', nm(mu64), 'nmse32', nm(mu32))
print('alpha64 quantiles', np.quantile(a64, [0, .1, .5, .9, .95, .99, 1]))
r = np.abs(a32-a64)/a64
print('per-coord rel alpha quantiles', np.quantile(r, [.5, .9, .99, 1]))
i = np.argsort(-a64)[:5]; print(a64[i], a32[i])
print('z support alpha64 max', a64[z!=0].max(), 'off-support min', a64[z==0].min())
