import numpy as np, sys
sys.path.insert(0, '.')
from oracle import cofem_oracle as O
g = np.load("tests/golden/multitask.npz")
def p2(m):
    return np.where(m > 0, 2.0 ** np.ceil(np.log2(np.where(m > 0, m, 1.0))), 1.0)
def oz_op(phi):
    phi = np.asarray(phi, np.float64)
    r = p2(np.abs(phi).max(axis=1)); c = p2((np.abs(phi) / r[:, None]).max(axis=0))
    phq = O.ozaki_dictionary(phi)
    def qcols(M, pre):
        X = M * pre[:, None]
        s = p2(np.abs(X).max(axis=0))
        return np.rint(X / s * 2.0**30) * s / 2.0**30 / pre[:, None]
    base = O.dense_op(phq)
    return O.Op(base.n_rows, base.n_cols, lambda V: phq @ qcols(V, c), lambda U: phq.T @ qcols(U, r),
                base.col_sq_norms, base.materialize, "dense")
phis = [g[f"dense_phi{l}"].astype(np.float64) for l in range(3)]
ys = [g[f"dense_y{l}"] for l in range(3)]
cfg = O.CofemConfig(iterations=6, probes=12, seed=3, cg=O.CgConfig(max_steps=400, tolerance=1e-5))
for name, ops in [("exact", [O.dense_op(p) for p in phis]), ("phiq", [O.dense_op(O.ozaki_dictionary(p)) for p in phis]), ("full", [oz_op(p) for p in phis])]:
    a, e, d = O.run_cofem_multitask(ops, ys, 1e4, cfg, share_probes=True)
    print(name, [x["cg_steps"] for x in d], np.linalg.norm(a - g["dense_alpha"]) / np.linalg.norm(g["dense_alpha"]))
def oz_op2(phi, fb, bb):
    phi = np.asarray(phi, np.float64)
    r = p2(np.abs(phi).max(axis=1)); c = p2((np.abs(phi) / r[:, None]).max(axis=0))
    phq = O.ozaki_dictionary(phi)
    def qcols(M, pre, bits):
        if bits is None: return M
        X = M * pre[:, None]
        s = p2(np.abs(X).max(axis=0))
        return np.rint(X / s * 2.0**bits) * s / 2.0**bits / pre[:, None]
    base = O.dense_op(phq)
    return O.Op(base.n_rows, base.n_cols, lambda V: phq @ qcols(V, c, fb), lambda U: phq.T @ qcols(U, r, bb),
                base.col_sq_norms, base.materialize, "dense")
for fb, bb in [(30, None), (None, 30), (38, 30), (30, 38), (46, 46)]:
    a, e, d = O.run_cofem_multitask([oz_op2(p, fb, bb) for p in phis], ys, 1e4, cfg, share_probes=True)
    print(fb, bb, [x["cg_steps"] for x in d])
