import sys, time, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2105_10439_b200 import _lib
rng = np.random.default_rng(0)
rel = lambda a, b: np.linalg.norm(a-b)/np.linalg.norm(b)
for (N, D, q) in [(256, 1024, 21), (100, 300, 5), (64, 1000, 40), (1, 7, 1), (513, 257, 33), (4096, 16384, 21)]:
    phi = (rng.standard_normal((N, D)) / np.sqrt(N)).astype(np.float32)
    ctx = _lib.Context(N, D, _lib.OZAKI); ctx.set_dictionary(phi)
    p64 = phi.astype(np.float64)
    V = rng.standard_normal((D, q)); U = rng.standard_normal((N, q))
    alpha = rng.random(D) + 0.5
    ref = 7.0 * p64.T @ (p64 @ V) + alpha[:, None] * V
    print(N, D, q, 'apply %.2e adj %.2e sys %.2e' % (rel(ctx.apply(V), p64 @ V), rel(ctx.apply_adjoint(U), p64.T @ U), rel(ctx.system_apply(7.0, alpha, V), ref)), flush=True)
    ctx.close()
