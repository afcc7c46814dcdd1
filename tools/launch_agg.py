"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"]
    m = re.search(r"(lob_\w+|dmma_gemm_v\d_kernel|dmma_gemm_kernel|splitk_reduce|perm_\w+|\w+_kernel)", name)
    key = m.group(1) if m else name[:40]
    v = float(d["Metric Value"].replace(",", ""))
    unit = d["Metric Unit"]
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    v *= scale.get(unit, 1.0)   # -> microseconds
    agg[key][0] += 1
    agg[key][1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v[1] / 1e3:9.3f} ms {100 * v[1] / tot:5.1f}%  n={v[0]:4d}  {k}")
print(f"total {tot / 1e3:.3f} ms")
