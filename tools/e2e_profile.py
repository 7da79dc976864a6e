"""Where the host time of run_cofem goes (context creation vs the run) on a structured config."""
import cProfile, io, os, pstats, sys, time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2105_10439_b200 import run_cofem
from paper_2105_10439_b200 import simulate as S

name = sys.argv[1] if len(sys.argv) > 1 else "dct-large"
if name in S.DCT_CONFIGS:
    c = S.DCT_CONFIGS[name]; prob, z = S.dct2_problem(c)
elif name in S.CONV_CONFIGS:
    c = S.CONV_CONFIGS[name]; prob, z = S.conv_problem(c)
else:
    c = S.CONFIGS[name]; prob, z, _ = S.dense_cs_problem(c)
cfg = c.cofem_config("auto", iterations=20)
run_cofem(prob, c.cofem_config("auto", iterations=2)); prob.op.release()   # warm the library
for rep in range(2):
    t0 = time.perf_counter(); ctx = prob.op.context(prob.op.resolve_precision("auto")); t1 = time.perf_counter()
    st, est, diag = run_cofem(prob, cfg); t2 = time.perf_counter()
    prob.op.release(); t3 = time.perf_counter()
    print(f"{name} rep {rep}: context {t1 - t0:.3f} s, run_cofem {t2 - t1:.3f} s ({20 / (t2 - t1):.2f} EM it/s), "
          f"device wall {sum(d['wall_time'] for d in diag):.3f} s, release {t3 - t2:.3f} s")
pr = cProfile.Profile(); pr.enable(); run_cofem(prob, cfg); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(18); print(s.getvalue()[:3500])
