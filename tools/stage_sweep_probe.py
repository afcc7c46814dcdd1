"""Per-stage tile / split-K sweep of one interface update (tt_debug_set_variant: tile id
v % 100, split v / 100), traced back-to-back (median of 7).  Shape args: a b al be [n]."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402

a, b, al, be = (int(v) for v in sys.argv[1:5]) if len(sys.argv) > 4 else (128, 128, 25, 25)
n = int(sys.argv[5]) if len(sys.argv) > 5 else 4
g = torch.Generator(device="cuda").manual_seed(0)
r = lambda *s: torch.randn(*s, dtype=torch.float64, device="cuda", generator=g)
phi, A, x = r(a, al, a), r(al, n, n, be), r(a, n, b)
out = torch.empty(b, be, b, dtype=torch.float64, device="cuda")
ws = torch.empty(tt.tt_interface_workspace_size(a, n, b, al, be), dtype=torch.uint8, device="cuda")
tt.tt_set_graph_cache(False)
ids = [10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21, 22, 24, 26, 29, 31]


def run(v):
    tt.tt_debug_set_variant(v)
    for _ in range(3):
        tt.tt_interface_left(phi, A, x, out, workspace=ws)
    torch.cuda.synchronize()
    tt.tt_trace_enable(200)
    for _ in range(7):
        tt.tt_interface_left(phi, A, x, out, workspace=ws)
    torch.cuda.synchronize()
    recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
    tt.tt_trace_disable()
    st = {}
    for rec in recs:
        st.setdefault(rec["stage"], []).append(rec["ms"] * 1e3)
    return {k: statistics.median(v) for k, v in st.items()}


base = run(-1)
print(f"shape a={a} b={b} al={al} be={be} n={n}; default: " +
      "  ".join(f"{k} {v:.1f}" for k, v in sorted(base.items())), flush=True)
best = {k: (v, -1) for k, v in base.items()}
for tid in ids:
    for ks in (1, 2, 4, 8):
        v = ks * 100 + tid if ks > 1 else tid
        try:
            t = run(v)
        except Exception as e:   # noqa: BLE001
            print("variant", v, "failed", e)
            continue
        for k, val in t.items():
            if val < best[k][0]:
                best[k] = (val, v)
tt.tt_debug_set_variant(-1)
print("best: " + "  ".join(f"{k} {v:.1f} us (variant {w})" for k, (v, w) in sorted(best.items())), flush=True)
