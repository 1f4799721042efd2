"""Average FSP_LB_PROF phase shares of the B&B's bounding launches (run with
FSP_LB_PROF=1; every launch prints one line on stderr)."""
import re
import sys
tot = {}
cnt = 0
for line in sys.stdin:
    if not line.startswith("FSP_LB_PROF"):
        continue
    cyc = float(re.search(r"\(([0-9.e+]+) warp-cycles\)", line).group(1))
    for name, pct in re.findall(r"(\w+) ([0-9.]+)%", line):
        tot[name] = tot.get(name, 0.0) + float(pct) * cyc / 100
    cnt += 1
s = sum(tot.values()) or 1
print(f"{cnt} launches:", " ".join(f"{k} {100 * v / s:.1f}%" for k, v in tot.items()))
