"""Share of each kernel in one bench step from an `ncu --metrics gpu__time_duration.sum` CSV.
The last `--per-step` launches of the library's kernels form the timed step."""
import csv
import re
import sys
from collections import OrderedDict


def main(path, per_step=None, skip=0):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.reader(lines)
    hdr = next(rd)
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    for r in rd:
        name = r[ki]
        if not re.search(r"dmma_gemm|fused_s12|small_chain|apply_|perm_|set_one|splitk|prep_all|prep_core|transpose_core|swap_bonds", name):
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1e6 if r[ui] == "ns" else (v / 1e3 if r[ui] == "us" else v)
        rows.append((name, v))
    if per_step:
        rows = rows[skip:skip + per_step] if skip else rows[-per_step:]
    agg = OrderedDict()
    for name, ms in rows:
        short = re.sub(r"\(.*", "", name)
        short = re.sub(r"CUtensorMap_st, CUtensorMap_st, ", "", short)
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(v[1] for v in agg.values())
    print(f"launches={len(rows)} total_ms={tot:.3f}")
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{ms / tot:7.2%}  {ms:9.3f} ms  {n:4d} launches  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None,
         int(sys.argv[3]) if len(sys.argv) > 3 else 0)
