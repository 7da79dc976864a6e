import numpy as np, sys
sys.path.insert(0, '.')
g_ = np.load("tests/golden/reference_workloads.npz"); golden = lambda n: g_
from paper_2105_10439_b200 import *
from oracle import cofem_oracle as O
g = golden("reference_workloads.npz")
op = SubsampledDctOperator(1024, g["dct_mask"])
prob = SblProblem(g["dct_y"], op, float(g["dct_beta"]))
for T in (1, 2, 3):
  for prec in ("ozaki", "fp64"):
    cfg = CofemConfig(iterations=T, probes=20, seed=0, cg=CgConfig(precision=prec))
    st, est, diag = run_cofem(prob, cfg)
    ocfg = O.CofemConfig(iterations=T, probes=20, seed=0)
    oa, omu, os_, od = O.run_cofem(O.dct_op(1024, g["dct_mask"]), g["dct_y"], float(g["dct_beta"]), ocfg)
    r = lambda a,b: np.linalg.norm(a-b)/np.linalg.norm(b)
    print(T, prec, [d["cg_steps"] for d in diag], [d["cg_steps"] for d in od],
          "mu", r(est.mu, omu), "a", r(st.alpha, oa), "resid", [d["cg_residual"] for d in diag][-1], od[-1]["cg_residual"], flush=True)
