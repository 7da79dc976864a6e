import numpy as np, sys
sys.path.insert(0, '.')
from oracle import cofem_oracle as O
g = np.load("tests/golden/reference_workloads.npz")
from scipy.fft import idct
mask = np.sort(g["dct_mask"])
phi = idct(np.eye(1024), axis=0, norm="ortho")[mask, :]
def q(phi, bits):
    rs = 2.0 ** np.ceil(np.log2(np.abs(phi).max(axis=1, keepdims=True)))
    return np.round(phi / rs * 2.0**bits) / 2.0**bits * rs
for name, P in [("exact", phi), ("q31", q(phi, 31)), ("q40", q(phi, 40)), ("f32", phi.astype(np.float32).astype(np.float64))]:
    cfg = O.CofemConfig(iterations=3, probes=20, seed=0)
    a, mu, s, d = O.run_cofem(O.dense_op(P), g["dct_y"], float(g["dct_beta"]), cfg)
    print(name, [x["cg_steps"] for x in d], np.abs(P @ P.T - np.eye(P.shape[0])).max())
