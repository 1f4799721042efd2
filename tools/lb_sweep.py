"""Time fsp_lb_eval across configs / launch shapes (CUDA events, inputs in HBM)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_1208_3933_b200 import binding, inputs


def time_cfg(name, N, warps=None, reps=5):
    if os.environ.get("FSP_LB_NPL") == "0":
        os.environ.pop("FSP_LB_NPL")
    if warps:
        os.environ["FSP_LB_WARPS"] = str(warps)
    else:
        os.environ.pop("FSP_LB_WARPS", None)
    n, m, seed = inputs.TAILLARD_SEEDS[name]
    ptm = inputs.taillard(n, m, seed)
    pf, dp = inputs.pool_d1(n, N, inputs.pool_seed(name))
    inst = binding.Instance(ptm)
    d_pf = torch.from_numpy(pf.view(np.int16)).cuda()
    d_dp = torch.from_numpy(dp).cuda()
    out = torch.empty(N, dtype=torch.int32, device="cuda")
    for _ in range(2):
        inst.lb_eval(d_pf, d_dp, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        inst.lb_eval(d_pf, d_dp, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    info = inst.info
    return {"cfg": name, "N": N, "npl": info["nodes_per_lane"], "warps": info["warps_per_cta"],
            "groups": info["groups"],
            "ctas_per_sm": info["ctas_per_sm"], "smem": info["smem_bytes"], "ms": round(ms, 3),
            "Mbounds_s": round(N / ms / 1e3, 2)}


if __name__ == "__main__":
    cfgs = sys.argv[1:] or ["ta091"]
    for c in cfgs:
        name, N = (c.split(":") + ["1048576"])[:2]
        for npl in os.environ.get("SWEEP_NPL", "0").split(","):
            os.environ["FSP_LB_NPL"] = npl
            for w in ([int(x) for x in os.environ.get("SWEEP_WARPS", "0").split(",")]):
                try:
                    r = time_cfg(name, int(N), w)
                except Exception as ex:  # a shape that does not fit: skip
                    print(json.dumps({"cfg": name, "npl_env": int(npl), "warps_env": w,
                                      "error": str(ex)[:120]}), flush=True)
                    continue
                r["npl_env"] = int(npl)
                print(json.dumps(r), flush=True)
