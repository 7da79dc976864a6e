import numpy as np, sys, time
sys.path.insert(0, '.')
from paper_2105_10439_b200 import *
from paper_2105_10439_b200 import simulate as S
g = np.load("tests/golden/cofem_dense-mid_T3.npz")
c = S.CONFIGS["dense-mid"]
prob, z, phi = S.dense_cs_problem(c)
print("ref", list(g["cg_steps"]))
for prec in ("ozaki", "fp64", "fp32"):
    for T in (3, 30):
        cfg = CofemConfig(iterations=T, probes=c.K, seed=c.seed, cg=CgConfig(max_steps=c.U, tolerance=c.tol, precision=prec))
        t0 = time.time(); st, est, d = run_cofem(prob, cfg); t1 = time.time()
        print(prec, T, [x["cg_steps"] for x in d], "nmse", S.nmse(est.mu, z) if hasattr(S, "nmse") else None, f"{t1-t0:.2f}s", flush=True)
