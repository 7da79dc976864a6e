import numpy as np, sys
sys.path.insert(0, '.')
from oracle import cofem_oracle as O
def phi32(rng, n, d):
    return (rng.standard_normal((n, d), dtype=np.float32) * np.float32(1.0 / np.sqrt(n))).astype(np.float32)
for (n, d, tol, T) in [(96,384,1e-5,6),(128,256,1e-6,6),(128,256,1e-5,8),(160,320,1e-6,6)]:
    rng = np.random.default_rng(77)
    zs = np.zeros(d); zs[rng.choice(d, size=12, replace=False)] = 1.0
    phis, ys = [], []
    for l in range(3):
        phi = phi32(rng, n, d); z = zs * rng.standard_normal(d)
        ys.append(phi.astype(np.float64) @ z + 0.01 * rng.standard_normal(n)); phis.append(phi.astype(np.float64))
    cfg = O.CofemConfig(iterations=T, probes=12, seed=3, cg=O.CgConfig(max_steps=400, tolerance=tol))
    a, e, d0 = O.run_cofem_multitask([O.dense_op(p) for p in phis], ys, 1e4, cfg, share_probes=True)
    a2, e2, d1 = O.run_cofem_multitask([O.dense_op(O.ozaki_dictionary(p)) for p in phis], ys, 1e4, cfg, share_probes=True)
    r = np.linalg.norm(a-a2)/np.linalg.norm(a)
    print(n, d, tol, [x["cg_steps"] for x in d0], [x["cg_steps"] for x in d1], r)
