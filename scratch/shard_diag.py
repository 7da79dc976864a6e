import numpy as np, sys
sys.path.insert(0, "tests")
from conftest import golden
from paper_2105_10439_b200 import simulate as S, run_cofem
from paper_2105_10439_b200.distributed import run_cofem_threaded
g = golden("cofem_dense-mid_T3.npz")
c = S.CONFIGS["dense-mid"]
prob, z, _ = S.dense_cs_problem(c)
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
for prec in ["fp64", "ozaki"]:
    for it in [1, 3]:
        cfg = c.cofem_config(prec, iterations=it)
        st0, e0, d0 = run_cofem(prob, cfg)
        for w in [1, 2]:
            st, e, d = run_cofem_threaded(prob, cfg, devices=[0] * w)
            print(prec, "T", it, "world", w, "steps", [x["cg_steps"] for x in d], [x["cg_steps"] for x in d0],
                  "mu vs unsharded", rel(e.mu, e0.mu), "s vs unsharded", rel(e.s, e0.s), "alpha", rel(st.alpha, st0.alpha), flush=True)
        prob.op.release()
