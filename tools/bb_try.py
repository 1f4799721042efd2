"""Time-boxed device B&B runs on Taillard instances (diagnostics)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1208_3933_b200 import binding, inputs

for arg in sys.argv[1:]:
    name, ub, secs = arg.split(":")
    p = inputs.instance(name)
    inst = binding.Instance(p)
    threads = int(os.environ.get("BB_THREADS", "0"))
    if threads:
        rc, ms, perm, st = inst.bb_solve_hybrid(threads, int(ub), 0, float(secs))
    else:
        rc, ms, perm, st = inst.bb_solve(int(ub), 0, float(secs))
    st["nodes_per_s"] = st["bounded"] / max(st["wall_s"], 1e-9)
    keep = ("bounded", "iterations", "wall_s", "nodes_per_s")
    print(json.dumps({"instance": name, "threads": threads, "initial_ub": int(ub), "rc": rc,
                      "makespan": ms, **{k: st[k] for k in keep}}),
          flush=True)
