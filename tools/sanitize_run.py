"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
LB pools exercising 1 and several couple groups, both walks (s16 / int32),
2 and 4 nodes per lane, ragged tails, malformed nodes; a small device B&B."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_1208_3933_b200 import binding, inputs


def run(name, N, **env):
    for k, v in env.items():
        os.environ[k] = str(v)
    n, m, seed = inputs.TAILLARD_SEEDS[name]
    p = inputs.taillard(n, m, seed)
    inst = binding.Instance(p)
    pf, dp = inputs.pool_d1(n, N, 5)
    out = inst.lb_eval(torch.from_numpy(pf.view(np.int16)).cuda(), torch.from_numpy(dp).cuda())
    torch.cuda.synchronize()
    assert inst.check() == binding.FSP_OK
    bad = pf.copy()
    bad[3, 0] = n + 7
    dp2 = dp.copy()
    dp2[3] = max(1, dp2[3])
    inst.lb_eval(torch.from_numpy(bad.view(np.int16)).cuda(), torch.from_numpy(dp2).cuda())
    torch.cuda.synchronize()
    assert inst.check() == binding.FSP_EBADNODE
    for k in env:
        os.environ.pop(k)
    print(name, N, inst.info, int(out.sum().item()), flush=True)


run("ta001", 1000)
run("ta021", 777, FSP_LB_NPL=4)
run("ta051", 333, FSP_LB_WARPS=4)
run("ta091", 301)
run("ta111", 129)
rng = np.random.default_rng(1)
p = rng.integers(1, 50, (8, 4)).astype(np.int32)
print(binding.Instance(p).bb_solve()[:2], flush=True)
print("sanitize workload done")
