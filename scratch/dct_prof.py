import sys, numpy as np
sys.path.insert(0, '.')
from paper_2105_10439_b200 import simulate as S, SystemMatrix
c = S.DCT_CONFIGS['dct-large']
prob, z = S.dct2_problem(c)
V = np.random.default_rng(0).standard_normal((c.D, 21))
for _ in range(2):
    out = SystemMatrix(prob.op, c.beta, np.ones(c.D)).apply(V)
print('ok', out.shape)
