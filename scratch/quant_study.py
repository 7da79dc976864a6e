import sys, time, numpy as np
sys.path.insert(0, '.')
from oracle import cofem_oracle as O
from paper_2105_10439_b200 import simulate as S
rel = lambda a, b: np.linalg.norm(a-b)/np.linalg.norm(b)

def pow2_scales(phi):
    # row scale r_i and col scale c_j, powers of two, so |phi/(r c)| <= 1
    a = np.abs(phi)
    r = 2.0 ** np.ceil(np.log2(a.max(axis=1) + 1e-300))
    a2 = a / r[:, None]
    c = 2.0 ** np.ceil(np.log2(a2.max(axis=0) + 1e-300))
    return r, c

def quant(x, bits):  # x in [-1, 1] -> fixed point with `bits` fractional bits (truncate toward -inf like 2's complement)
    s = 2.0 ** bits
    return np.floor(x * s) / s

def make_apply(phi, beta, alpha, F, G):
    r, c = pow2_scales(phi)
    ph = quant(phi / r[:, None] / c[None, :], F) * r[:, None] * c[None, :]
    def qcols(M):
        m = np.abs(M).max(axis=0); e = 2.0 ** np.ceil(np.log2(m + 1e-300)); e[m == 0] = 1
        return quant(M / e, G) * e
    def fn(V):
        U = ph @ qcols(V)
        return beta * (ph.T @ qcols(U)) + alpha[:, None] * V
    return fn

def run(phi, y, beta, cfg, F, G, T):
    rng = O.substream(cfg.seed, 3)
    D = phi.shape[1]; alpha = np.ones(D); op = O.dense_op(phi)
    aty = op.adjoint(y[:, None])
    for t in range(T):
        probes = O.draw_rademacher(D, cfg.probes, rng)
        rhs = np.concatenate([probes, aty], axis=1)
        minv = 1.0 / (beta + alpha)
        rep = O.pcg_solve(make_apply(phi, beta, alpha, F, G), rhs, minv, cfg.cg)
        mu = beta * rep.solution[:, cfg.probes]; s = (probes * rep.solution[:, :cfg.probes]).mean(axis=1)
        if t < T - 1: alpha = O.m_step(mu, s)
    return alpha, mu

for name, gname, T in [('dense-small', 'cofem_dense-small.npz', 50), ('dense-mid', 'cofem_dense-mid_T3.npz', 3)]:
    if len(sys.argv) > 1 and name not in sys.argv[1:]: continue
    g = np.load('tests/golden/' + gname)
    c = S.CONFIGS[name]
    phi = S.gaussian_dictionary(c.N, c.D, c.seed).astype(np.float64)
    cfg = O.CofemConfig(iterations=T, probes=c.K, seed=c.seed, cg=O.CgConfig(max_steps=c.U, tolerance=c.tol))
    for F, G in [(24, 24), (31, 31), (36, 36), (40, 40), (48, 48)]:
        t = time.time(); a, mu = run(phi, g['y'], c.beta, cfg, F, G, T)
        print(name, F, G, 'mu %.2e alpha %.2e' % (rel(mu, g['mu']), rel(a, g['alpha'])), '%.0fs' % (time.time() - t), flush=True)
