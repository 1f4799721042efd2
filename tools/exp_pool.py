"""Runtime pool-size choice (fsp_lb_tune_pool) per config, and the B&B's
nodes/s and incumbent for several per-iteration child caps."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1208_3933_b200 import binding, inputs  # noqa: E402

if sys.argv[1:2] == ["tune"]:
    for cfg in ("ta001", "ta021", "ta051", "ta091", "ta111"):
        inst = binding.Instance(inputs.instance(cfg))
        pool, rates = inst.tune_pool(22, 0.95)
        print(json.dumps({"instance": cfg, "pool_95": pool,
                          "rates": {str(k): round(v / 1e6, 1) for k, v in rates.items()}}), flush=True)
else:
    for cap in sys.argv[1:]:
        env = dict(os.environ, FSP_BB_CHILDREN=cap)
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bb_try.py"),
                              "ta051:2147483647:10", "ta091:2147483647:10"], env=env,
                             capture_output=True, text=True).stdout
        for line in out.splitlines():
            d = json.loads(line)
            print(json.dumps({"cap": int(cap), "instance": d["instance"], "incumbent": d["makespan"],
                              "nodes_per_s": round(d["nodes_per_s"] / 1e6, 1),
                              "iterations": d["iterations"]}), flush=True)
