import time, numpy as np
from paper_2105_10439_b200 import _lib
from paper_2105_10439_b200 import simulate as S
c = S.CONFIGS["dense-large"]
phi = S.gaussian_dictionary(c.N, c.D, c.seed)
import torch; torch.cuda.init()
for rep in range(2):
    t0 = time.perf_counter(); ctx = _lib.Context(c.N, c.D, _lib.OZAKI, 0); t1 = time.perf_counter()
    ctx.set_dictionary(phi); t2 = time.perf_counter()
    ctx.apply(np.zeros((c.D, 1))); t3 = time.perf_counter()
    ctx.close(); t4 = time.perf_counter()
    print(f"create {t1-t0:.3f}s set_dictionary {t2-t1:.3f}s ({phi.nbytes/(t2-t1)/1e9:.1f} GB/s) planes+apply {t3-t2:.3f}s close {t4-t3:.3f}s", flush=True)
