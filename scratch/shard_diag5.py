import numpy as np
from paper_2105_10439_b200 import DenseOperator
from paper_2105_10439_b200 import simulate as S
from paper_2105_10439_b200.distributed import threaded_contexts, run_threaded
c = S.CONFIGS["dense-mid"]
prob, z, _ = S.dense_cs_problem(c)
op = prob.op; phi = op.matrix
y = np.asarray(prob.y)[:, None]
ref = phi.astype(np.float64).T @ y
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
print("unsharded aty", rel(op.context("ozaki").apply_adjoint(y), ref))
ctxs, sh = threaded_contexts(op, "ozaki", [0, 0])
a = run_threaded(2, lambda r: ctxs[r].apply_adjoint(y), ctxs[0].group)
print("sharded aty", rel(np.concatenate(a), ref))
Y8 = np.repeat(y, 8, axis=1) * np.arange(1, 9)
print("unsharded 8", rel(op.context("ozaki").apply_adjoint(Y8), phi.astype(np.float64).T @ Y8))
a = run_threaded(2, lambda r: ctxs[r].apply_adjoint(Y8), ctxs[0].group)
print("sharded 8", rel(np.concatenate(a), phi.astype(np.float64).T @ Y8))
