import os, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1208_3933_b200 import binding, inputs
name = sys.argv[1]; N = int(sys.argv[2])
n, m, seed = inputs.TAILLARD_SEEDS[name]
pf, dp = inputs.pool_d1(n, N, 99)
inst = binding.Instance(inputs.taillard(n, m, seed))
print(inst.launch_info(N), flush=True)
out = inst.lb_eval(torch.from_numpy(pf.view(np.int16)).cuda(), torch.from_numpy(dp).cuda())
torch.cuda.synchronize()
print("done", out[:4].tolist(), flush=True)
