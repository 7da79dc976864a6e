import numpy as np
from paper_2105_10439_b200 import DenseOperator
from paper_2105_10439_b200.distributed import threaded_contexts, run_threaded
rng = np.random.default_rng(0)
n, d, q = 1024, 4096, 21
phi = (rng.standard_normal((n, d)) / np.sqrt(n)).astype(np.float32)
op = DenseOperator(phi)
B = rng.standard_normal((d, q)); alpha = rng.random(d) + 0.5; beta = 1e4
minv = 1.0 / (beta + alpha)
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
ref = op.context("fp64").pcg_solve(beta, alpha, minv, B, 12, 1e-30)[0]
full = op.context("ozaki").pcg_solve(beta, alpha, minv, B, 12, 1e-30)[0]
print("unsharded ozaki vs fp64", rel(full, ref))
for prec in ["fp64", "ozaki"]:
    for w in [2]:
        ctxs, sh = threaded_contexts(op, prec, [0] * w)
        X = run_threaded(w, lambda r: ctxs[r].pcg_solve(beta, alpha[sh[r][0]:sh[r][1]], minv[sh[r][0]:sh[r][1]],
                         np.ascontiguousarray(B[sh[r][0]:sh[r][1]]), 12, 1e-30)[0], ctxs[0].group)
        print(prec, "world", w, "vs fp64", rel(np.concatenate(X), ref))
        for c in ctxs: c.close()
