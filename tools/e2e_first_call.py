"""bench.py's e2e region for a structured config: the FIRST run_cofem of the process, profiled."""
import cProfile, io, os, pstats, sys, time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2105_10439_b200 import run_cofem
from paper_2105_10439_b200 import simulate as S

name = sys.argv[1] if len(sys.argv) > 1 else "dct-large"
c = S.DCT_CONFIGS[name] if name in S.DCT_CONFIGS else S.CONV_CONFIGS[name]
prob, z = S.dct2_problem(c) if name in S.DCT_CONFIGS else S.conv_problem(c)
ctx = prob.op.context("ozaki")
ctx.bench_prepare(np.asarray(prob.y), c.beta, c.K, c.U, c.tol, seed=1)
ctx.bench_iterations(2)
prob.op.release()
cfg = c.cofem_config("ozaki", iterations=20)
pr = cProfile.Profile(); t0 = time.perf_counter(); pr.enable(); run_cofem(prob, cfg); pr.disable(); el = time.perf_counter() - t0
print(f"{name}: first run_cofem {el:.3f} s = {20 / el:.2f} EM it/s")
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(14); print(s.getvalue()[:3000])
