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
# round 2: B&B with ordering / dive / unscheduled lists (ta091 few iterations),
# the family kernel, the hybrid solver, the pinned-host gather path
os.environ["FSP_BB_CHILDREN"] = "8192"
os.environ["FSP_BB_MEM_FRAC"] = "0.02"
inst = binding.Instance(inputs.instance("ta091"))
bb = binding.BBState(inst)
bb.step(12)
print("bb ta091", bb.stats()["bounded"], flush=True)
bb.close()
i20 = binding.Instance(inputs.instance("ta021"))
pf, dp = inputs.pool_fixed_depth(20, 64, 8, 3)
print("family", int(i20.lb_eval_children(torch.from_numpy(pf.view(np.int16)).cuda(),
                                        torch.from_numpy(dp).cuda()).sum().item()), flush=True)
print("hybrid", binding.Instance(p).bb_solve_hybrid(2)[:2], flush=True)
n = 200
pf, dp = inputs.pool_d1(n, 148 * 16 * 128 + 77, 9)
h_pf = torch.from_numpy(pf.view(np.int16)).pin_memory()
h_dp = torch.from_numpy(dp).pin_memory()
h_lb = torch.empty(len(dp), dtype=torch.int32).pin_memory()
inst.lb_eval_host_ptr(h_pf.data_ptr(), pf.shape[1], h_dp.data_ptr(), len(dp), h_lb.data_ptr())
print("host gather", int(h_lb.sum().item()), flush=True)
# round 2b: the warp-per-sub-problem A/B kernel (wpn.cu)
os.environ["FSP_LB_MAPPING"] = "warp"
iw = binding.Instance(inputs.instance("ta021"))
pf, dp = inputs.pool_d1(20, 301, 4)
print("wpn", int(iw.lb_eval(torch.from_numpy(pf.view(np.int16)).cuda(), torch.from_numpy(dp).cuda()).sum().item()),
      flush=True)
os.environ.pop("FSP_LB_MAPPING")
print("sanitize workload done")
