import numpy as np, sys
sys.path.insert(0, '.')
from paper_2105_10439_b200 import *
from oracle import cofem_oracle as O
g = np.load("tests/golden/conv_cases.npz")
prob = SblProblem(g["y"], build_exp_convolution(512, 0.04), float(g["beta"]))
for K in (20, 31, 32, 40):
    for prec in ("ozaki",):
        cfg = CofemConfig(iterations=3, probes=K, seed=4, cg=CgConfig(max_steps=400, tolerance=1e-6, precision=prec))
        st, est, diag = run_cofem(prob, cfg)
        ocfg = O.CofemConfig(iterations=3, probes=K, seed=4, cg=O.CgConfig(max_steps=400, tolerance=1e-6))
        a, mu, s, od = O.run_cofem(O.conv_op(512, (1.0 - 0.04) ** np.arange(512, dtype=np.float64)), g["y"], float(g["beta"]), ocfg)
        print(K, prec, [d["cg_steps"] for d in diag], [d["cg_steps"] for d in od], np.linalg.norm(est.mu-mu)/np.linalg.norm(mu), flush=True)
