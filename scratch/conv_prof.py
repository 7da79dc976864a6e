import sys, numpy as np
sys.path.insert(0, '.')
from paper_2105_10439_b200 import _lib, simulate as S
c = S.CONV_CONFIGS['conv-large']
h = c.taps()
ctx = _lib.Context.convolution(c.D, h, _lib.OZAKI, 0)
V = np.random.default_rng(0).standard_normal((c.D, 31))
for _ in range(2):
    out = ctx.system_apply(c.beta, np.ones(c.D), V)
print('ok', out.shape)
