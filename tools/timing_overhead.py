"""Does per-kernel event timing (bench.py's time_kernels=True) slow the
device-timed total?  Runs each structured config's EM iterations with and
without the per-launch CUDA events, alternating."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2105_10439_b200 import simulate as S

which = sys.argv[1] if len(sys.argv) > 1 else "dct-large"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if which in S.DCT_CONFIGS:
    c = S.DCT_CONFIGS[which]; prob, z = S.dct2_problem(c)
else:
    c = S.CONV_CONFIGS[which]; prob, z = S.conv_problem(c)
ctx = prob.op.context("auto")
y = np.asarray(prob.y)
for rep in range(2):
    for tk in (False, True):
        ctx.bench_prepare(y, c.beta, c.K, c.U, c.tol, seed=0xC0FE)
        t = ctx.bench_iterations(T, time_kernels=tk)
        print(which, "time_kernels", tk, "total_ms %.2f" % t["total_ms"], "pcg", t["pcg_steps"],
              "ms/step %.4f" % (t["total_ms"] / t["pcg_steps"]), "fwd_ms %.3f" % t["fwd_ms"], flush=True)
