import time, numpy as np
from paper_2105_10439_b200 import run_cofem
from paper_2105_10439_b200 import simulate as S
c = S.DCT_CONFIGS["dct-large"]
prob, z = S.dct2_problem(c)
for rep in range(3):
    cfg = c.cofem_config("ozaki", iterations=20)
    t0 = time.perf_counter(); ctx = prob.op.context("ozaki"); t1 = time.perf_counter()
    st, est, diag = run_cofem(prob, cfg); t2 = time.perf_counter()
    st, est, diag = run_cofem(prob, cfg); t3 = time.perf_counter()
    prob.op.release(); t4 = time.perf_counter()
    print(f"create {t1-t0:.3f} first run {t2-t1:.3f} second run {t3-t2:.3f} release {t4-t3:.3f}", flush=True)
