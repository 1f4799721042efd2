"""Per-kernel time shares of an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import re
import sys

for f in sys.argv[1:]:
    rows = list(csv.reader([l for l in open(f) if l.startswith('"')]))
    ix = {h: i for i, h in enumerate(rows[0])}
    agg, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        k = re.sub(r"\(.*", "", r[ix["Kernel Name"]]).replace("void ", "").replace("<unnamed>::", "")
        v = float(r[ix["Metric Value"]].replace(",", ""))
        u = r[ix["Metric Unit"]]
        v = v / 1000 if u == "ns" else (v * 1000 if u == "ms" else v)
        agg[k] += v
        cnt[k] += 1
    tot = sum(agg.values())
    print(f"{f}: {len(rows) - 1} launches, {tot / 1000:.2f} ms")
    for k, v in agg.most_common():
        print(f"  {k[:48]:48s} {cnt[k]:5d}  {100 * v / tot:5.1f} %  {v / cnt[k]:9.1f} us/launch")
