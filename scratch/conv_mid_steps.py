import numpy as np, sys, json
sys.path.insert(0, '.')
from paper_2105_10439_b200 import run_cofem
from paper_2105_10439_b200 import simulate as S
c = S.CONV_CONFIGS["conv-mid"]
prob, z = S.conv_problem(c)
st, est, diag = run_cofem(prob, c.cofem_config())
json.dump({"steps": [d["cg_steps"] for d in diag], "mu": est.mu.tolist()[:10]}, open("gpurun_out/conv_mid_gpu.json", "w"))
print([d["cg_steps"] for d in diag])
