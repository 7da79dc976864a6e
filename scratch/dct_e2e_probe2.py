import time, numpy as np
from paper_2105_10439_b200 import run_cofem
from paper_2105_10439_b200 import simulate as S
c = S.DCT_CONFIGS["dct-large"]
prob, z = S.dct2_problem(c)
ctx = prob.op.context("ozaki")
ctx.bench_prepare(np.asarray(prob.y), c.beta, c.K, c.U, c.tol, seed=0xC0FE)
ctx.bench_iterations(3)
ctx.bench_prepare(np.asarray(prob.y), c.beta, c.K, c.U, c.tol, seed=0xC0FE)
t = ctx.bench_iterations(20, time_kernels=True)
print("device", t["total_ms"], flush=True)
prob.op.release()
for rep in range(3):
    cfg = c.cofem_config("ozaki", iterations=20)
    t0 = time.perf_counter(); cx = prob.op.context("ozaki"); t1 = time.perf_counter()
    st, est, diag = run_cofem(prob, cfg); t2 = time.perf_counter()
    prob.op.release(); t3 = time.perf_counter()
    print(f"create {t1-t0:.3f} run {t2-t1:.3f} release {t3-t2:.3f} steps {sum(d['cg_steps'] for d in diag)}", flush=True)
