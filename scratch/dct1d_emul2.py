import numpy as np, sys
sys.path.insert(0, '.')
from oracle import cofem_oracle as O
g = np.load("tests/golden/reference_workloads.npz")
from scipy.fft import idct
mask = np.sort(g["dct_mask"])
phi = idct(np.eye(1024), axis=0, norm="ortho")[mask, :]
cfg = O.CofemConfig(iterations=30, probes=20, seed=0)
a, mu, s, d = O.run_cofem(O.dense_op(O.ozaki_dictionary(phi)), g["dct_y"], float(g["dct_beta"]), cfg)
print([x["cg_steps"] for x in d])
