import numpy as np
from paper_2105_10439_b200 import run_cofem
from paper_2105_10439_b200 import simulate as S
c = S.CONFIGS["dense-mid"]
prob, z, _ = S.dense_cs_problem(c)
for prec in ["fp64", "ozaki", "fp64", "ozaki"]:
    for rep in range(3):
        st, est, diag = run_cofem(prob, c.cofem_config(prec, iterations=1))
        print(prec, rep, [d["cg_steps"] for d in diag], float(np.linalg.norm(est.mu)), flush=True)
    prob.op.release()
