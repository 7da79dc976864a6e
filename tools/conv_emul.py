import numpy as np, sys
sys.path.insert(0, '.')
from oracle import cofem_oracle as O
g = np.load("tests/golden/conv_cases.npz")
h = (1.0 - 0.04) ** np.arange(512, dtype=np.float64)
def p2(m): return np.where(m > 0, 2.0 ** np.ceil(np.log2(np.where(m > 0, m, 1.0))), 1.0)
hs = p2(np.abs(h).max())
def qtaps(h, bits=30): return np.rint(h / hs * 2.0**bits) * hs / 2.0**bits
def qcols(M, bits=30):
    s = p2(np.abs(M).max(axis=0)); return np.rint(M / s * 2.0**bits) * s / 2.0**bits
def op_with(hh, qop):
    base = O.conv_op(512, hh)
    ap = (lambda V: base.apply(qcols(V))) if qop else base.apply
    ad = (lambda U: base.adjoint(qcols(U))) if qop else base.adjoint
    return O.Op(base.n_rows, base.n_cols, ap, ad, base.col_sq_norms, base.materialize, "conv")
cfg = O.CofemConfig(iterations=3, probes=20, seed=4, cg=O.CgConfig(max_steps=400, tolerance=1e-6))
for name, hh, qop in [("exact", h, False), ("taps31", qtaps(h), False), ("operand31", h, True), ("both", qtaps(h), True),
                      ("operand38", h, "38")]:
    if qop == "38":
        base = O.conv_op(512, hh)
        op = O.Op(512, 512, lambda V: base.apply(qcols(V, 37)), lambda U: base.adjoint(qcols(U, 37)), base.col_sq_norms, base.materialize, "conv")
    else:
        op = op_with(hh, qop)
    a, mu, s, d = O.run_cofem(op, g["y"], float(g["beta"]), cfg)
    print(name, [x["cg_steps"] for x in d])
def qrel(M, bits=31):
    m, e = np.frexp(M); return np.ldexp(np.rint(m * 2.0**bits) / 2.0**bits, e)
for name, f in [("relative31", qrel), ("relative24", lambda M: qrel(M, 24))]:
    base = O.conv_op(512, h)
    op = O.Op(512, 512, lambda V, f=f: base.apply(f(V)), lambda U, f=f: base.adjoint(f(U)), base.col_sq_norms, base.materialize, "conv")
    a, mu, s, d = O.run_cofem(op, g["y"], float(g["beta"]), cfg)
    print(name, [x["cg_steps"] for x in d])
print("beta", float(g["beta"]))
