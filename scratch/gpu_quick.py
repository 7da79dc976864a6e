import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_2105_10439_b200 import _lib
from paper_2105_10439_b200 import simulate as S
from oracle import cofem_oracle as O
print('devices', _lib.device_count())
rng = np.random.default_rng(0)
for prec in (_lib.FP64, _lib.FP32):
    for (N, D, q) in [(256, 1024, 21), (100, 300, 5), (64, 1000, 40)]:
        phi = rng.standard_normal((N, D)).astype(np.float32)
        ctx = _lib.Context(N, D, prec)
        ctx.set_dictionary(phi)
        V = rng.standard_normal((D, q)); U = rng.standard_normal((N, q))
        p64 = phi.astype(np.float64)
        r1 = np.linalg.norm(ctx.apply(V) - p64 @ V) / np.linalg.norm(p64 @ V)
        r2 = np.linalg.norm(ctx.apply_adjoint(U) - p64.T @ U) / np.linalg.norm(p64.T @ U)
        alpha = rng.random(D) + 0.5
        ref = 3.0 * p64.T @ (p64 @ V) + alpha[:, None] * V
        r3 = np.linalg.norm(ctx.system_apply(3.0, alpha, V) - ref) / np.linalg.norm(ref)
        print(prec, N, D, q, 'apply %.2e adj %.2e sys %.2e' % (r1, r2, r3))
        ctx.close()
cfg = S.CONFIGS['dense-small']
prob, z, phi = S.dense_cs_problem(cfg)
op = O.dense_op(phi)
ocfg = O.CofemConfig(iterations=cfg.T, probes=cfg.K, cg=O.CgConfig(max_steps=cfg.U, tolerance=cfg.tol))
from paper_2105_10439_b200.cofem import draw_probe_blocks, run_cofem
pb = draw_probe_blocks(cfg.D, cfg.K, cfg.T, cfg.seed)
t=time.time(); a64, mu64, s64, d64 = O.run_cofem(op, prob.y, cfg.beta, ocfg); print('oracle', time.time()-t)
rel = lambda a,b: np.linalg.norm(a-b)/np.linalg.norm(b)
for prec in ('fp64', 'fp32'):
    t=time.time(); st, est, diag = run_cofem(prob, cfg.cofem_config(prec)); el=time.time()-t
    print(prec, 'time %.2f' % el, 'rel mu %.2e alpha %.2e s %.2e' % (rel(est.mu, mu64), rel(st.alpha, a64), rel(est.s, s64)))
    print(' steps', [d['cg_steps'] for d in diag][:8], [d['cg_steps'] for d in d64][:8])
    print(' nmse', S.nmse(est.mu, z), S.nmse(mu64, z))
