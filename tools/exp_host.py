"""fsp_lb_eval_host timing on pinned buffers (e2e leg of bench.py) for
chunk sizes / gather SM counts given as env overrides on the command line."""
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 1 and sys.argv[1] == "run":
    import numpy as np
    import torch
    from paper_1208_3933_b200 import binding, inputs
    n, m, seed = inputs.TAILLARD_SEEDS["ta091"]
    N = 1 << 20
    pf, dp = inputs.pool_d1(n, N, inputs.pool_seed("ta091"))
    inst = binding.Instance(inputs.taillard(n, m, seed))
    h_pf = torch.from_numpy(pf.view(np.int16)).pin_memory()
    h_dp = torch.from_numpy(dp).pin_memory()
    h_lb = torch.empty(N, dtype=torch.int32).pin_memory()
    for _ in range(2):
        inst.lb_eval_host_ptr(h_pf.data_ptr(), pf.shape[1], h_dp.data_ptr(), N, h_lb.data_ptr())
    t0 = time.perf_counter()
    for _ in range(10):
        inst.lb_eval_host_ptr(h_pf.data_ptr(), pf.shape[1], h_dp.data_ptr(), N, h_lb.data_ptr())
    dt = (time.perf_counter() - t0) / 10
    print(f"{os.environ.get('TAG', '')}: {dt * 1e3:.2f} ms/step, e2e {N / dt:.4g} bounds/s", flush=True)
    sys.exit(0)
for spec in sys.argv[1:]:
    env = dict(os.environ, TAG=spec)
    for kv in spec.split(","):
        if kv:
            k, v = kv.split("=")
            env[k] = v
    subprocess.run([sys.executable, __file__, "run"], env=env)
