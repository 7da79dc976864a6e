import numpy as np
from paper_2105_10439_b200 import DenseOperator
from paper_2105_10439_b200.distributed import threaded_contexts, run_threaded
rng = np.random.default_rng(0)
n, d, q = 1024, 4096, 21
A = (rng.standard_normal((n, d // 2)) / np.sqrt(n)).astype(np.float32)
for name, phi in [("random", (rng.standard_normal((n, d)) / np.sqrt(n)).astype(np.float32)), ("[A A]", np.concatenate([A, A], 1))]:
    op = DenseOperator(phi)
    B = rng.standard_normal((d, q)); alpha = rng.random(d) + 0.5; beta = 1e4
    minv = 1.0 / (beta + alpha)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    for steps in [1, 2, 4, 12]:
        ref = op.context("fp64").pcg_solve(beta, alpha, minv, B, steps, 1e-30)[0]
        full = op.context("ozaki").pcg_solve(beta, alpha, minv, B, steps, 1e-30)[0]
        ctxs, sh = threaded_contexts(op, "ozaki", [0, 0])
        X = run_threaded(2, lambda r: ctxs[r].pcg_solve(beta, alpha[sh[r][0]:sh[r][1]], minv[sh[r][0]:sh[r][1]],
                         np.ascontiguousarray(B[sh[r][0]:sh[r][1]]), steps, 1e-30)[0], ctxs[0].group)
        Xs = np.concatenate(X)
        print(name, "steps", steps, "unsharded", rel(full, ref), "sharded", rel(Xs, ref), "percol", np.round(np.linalg.norm(Xs - ref, axis=0) / np.linalg.norm(ref, axis=0) * 1e9, 2)[:6], flush=True)
        for c in ctxs: c.close()
    op.release()
