"""Per-phase cycle shares of the bounding kernel (FSP_LB_PROF=1 makes every
launch record clock64 deltas per warp: ingest, heads, group wait, walk,
buffer release, store) and the plain launch time, per config.
usage: python tools/lb_prof.py ta091:1048576 [ta111:262144 ...]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1208_3933_b200 import binding, inputs  # noqa: E402

for arg in sys.argv[1:]:
    name, N = arg.split(":")
    N = int(N)
    n, m, seed = inputs.TAILLARD_SEEDS[name]
    ptm = inputs.taillard(n, m, seed)
    pf, dp = inputs.pool_d1(n, N, inputs.pool_seed(name) if name in inputs.CONFIGS else 5)
    inst = binding.Instance(ptm)
    d_pf = torch.from_numpy(pf.view(np.int16)).cuda()
    d_dp = torch.from_numpy(dp).cuda()
    out = torch.empty(N, dtype=torch.int32, device="cuda")
    for _ in range(3):
        inst.lb_eval(d_pf, d_dp, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10):
        inst.lb_eval(d_pf, d_dp, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name} {n}x{m} pool {N}: {ms:.3f} ms, {N / ms / 1e3:.4g} bounds/s, launch "
          f"{inst.launch_info(N)}", flush=True)
    os.environ["FSP_LB_PROF"] = "1"
    inst.lb_eval(d_pf, d_dp, out)
    torch.cuda.synchronize()
    del os.environ["FSP_LB_PROF"]
