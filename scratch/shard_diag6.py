import numpy as np, sys
from oracle import cofem_oracle as O
from paper_2105_10439_b200 import simulate as S, run_cofem
from paper_2105_10439_b200.distributed import run_cofem_threaded
c = S.CONFIGS["dense-mid"]
prob, z, _ = S.dense_cs_problem(c)
phi = prob.op.matrix
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
for T in [1, 2]:
    ocfg = O.CofemConfig(iterations=T, probes=c.K, seed=c.seed, cg=O.CgConfig(max_steps=c.U, tolerance=c.tol))
    alpha, mu, s, od = O.run_cofem(O.dense_op(phi), np.asarray(prob.y), c.beta, ocfg)
    for prec in ["fp64", "ozaki"]:
        cfg = c.cofem_config(prec, iterations=T)
        st0, e0, d0 = run_cofem(prob, cfg)
        st1, e1, d1 = run_cofem_threaded(prob, cfg, devices=[0, 0])
        print("T", T, prec, "oracle steps", [d["cg_steps"] for d in od], "unsharded", [d["cg_steps"] for d in d0], rel(e0.mu, mu), rel(e0.s, s),
              "| sharded", [d["cg_steps"] for d in d1], rel(e1.mu, mu), rel(e1.s, s), flush=True)
        prob.op.release()
