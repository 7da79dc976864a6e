import numpy as np
from paper_2105_10439_b200 import DenseOperator
from paper_2105_10439_b200.distributed import threaded_contexts, run_threaded
rng = np.random.default_rng(0)
n, d, q = 1024, 4096, 21
phi = (rng.standard_normal((n, d)) / np.sqrt(n)).astype(np.float32)
op = DenseOperator(phi)
P = rng.standard_normal((d, q)); U = rng.standard_normal((n, q))
ref_f = phi.astype(np.float64) @ P; ref_a = phi.astype(np.float64).T @ U
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
full = op.context("ozaki")
print("unsharded fwd", rel(full.apply(P), ref_f), "adj", rel(full.apply_adjoint(U), ref_a))
for w in [2, 3]:
    ctxs, shards = threaded_contexts(op, "ozaki", [0] * w)
    f = run_threaded(w, lambda r: ctxs[r].apply(np.ascontiguousarray(P[shards[r][0]:shards[r][1]])), ctxs[0].group)
    a = run_threaded(w, lambda r: ctxs[r].apply_adjoint(U), ctxs[0].group)
    print("world", w, "fwd", [rel(x, ref_f) for x in f], "adj", rel(np.concatenate(a), ref_a))
    sysm = run_threaded(w, lambda r: ctxs[r].system_apply(1e4, np.ones(shards[r][1]-shards[r][0]), np.ascontiguousarray(P[shards[r][0]:shards[r][1]])), ctxs[0].group)
    ref_s = 1e4 * (phi.astype(np.float64).T @ ref_f) + P
    print("   system", rel(np.concatenate(sysm), ref_s), "unsharded", rel(full.system_apply(1e4, np.ones(d), P), ref_s))
    for c in ctxs: c.close()
