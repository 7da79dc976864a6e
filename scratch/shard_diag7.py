import numpy as np
from oracle import cofem_oracle as O
from paper_2105_10439_b200 import simulate as S
from paper_2105_10439_b200.distributed import threaded_contexts, run_threaded
c = S.CONFIGS["dense-mid"]
prob, z, _ = S.dense_cs_problem(c)
phi = prob.op.matrix; op = prob.op
probes = O.draw_rademacher(c.D, c.K, O.substream(c.seed, 3))
aty = phi.astype(np.float64).T @ np.asarray(prob.y)
B = np.concatenate([probes, aty[:, None]], 1)
P = B / (c.beta * 1.0 + 1.0)
alpha = np.ones(c.D)
ref = c.beta * (phi.astype(np.float64).T @ (phi.astype(np.float64) @ P)) + P
pc = lambda X: np.linalg.norm(X - ref, axis=0) / np.linalg.norm(ref, axis=0)
full = op.context("ozaki").system_apply(c.beta, alpha, P)
ctxs, sh = threaded_contexts(op, "ozaki", [0, 0])
Xs = np.concatenate(run_threaded(2, lambda r: ctxs[r].system_apply(c.beta, alpha[sh[r][0]:sh[r][1]], np.ascontiguousarray(P[sh[r][0]:sh[r][1]])), ctxs[0].group))
np.set_printoptions(precision=2)
print("norms", np.linalg.norm(P, axis=0)[[0, 1, -1]])
print("unsharded per-col err", pc(full)[[0, 1, 2, -2, -1]])
print("sharded   per-col err", pc(Xs)[[0, 1, 2, -2, -1]])
V = phi.astype(np.float64) @ P
print("V col norms", np.linalg.norm(V, axis=0)[[0, 1, -1]], "V col max", np.abs(V).max(0)[[0, 1, -1]])
for r in range(2):
    Vr = phi[:, sh[r][0]:sh[r][1]].astype(np.float64) @ P[sh[r][0]:sh[r][1]]
    print("rank", r, "partial V col norms", np.linalg.norm(Vr, axis=0)[[0, 1, -1]])
