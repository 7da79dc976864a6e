import numpy as np, sys
sys.path.insert(0, '.')
from paper_2105_10439_b200 import _lib
D = 1 << 22
taps = 0.98 ** np.arange(256)
ctx = _lib.Context.convolution(D, taps, _lib.OZAKI, 0)
V = np.random.default_rng(0).standard_normal((D, 31))
for _ in range(2):
    U = ctx.apply(V)
    W = ctx.apply_adjoint(U)
print("ok", float(np.abs(U).sum()) > 0)
