"""Interface update (left / right) at the config-5 interior-core shape, timed alone with the
library's event tracer: per-stage TFLOP/s (the W5 sweep runs them concurrently with the
matvecs, so their in-step numbers are not their own)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402

a = b = int(sys.argv[1]) if len(sys.argv) > 1 else 256
al = be = int(sys.argv[2]) if len(sys.argv) > 2 else 36
n = 4
g = torch.Generator(device="cuda").manual_seed(0)
r = lambda *s: torch.randn(*s, dtype=torch.float64, device="cuda", generator=g)
phiL, A, phiR, x = r(a, al, a), r(al, n, n, be), r(b, be, b), r(a, n, b)
wi = torch.empty(tt.tt_interface_workspace_size(a, n, b, al, be), dtype=torch.uint8, device="cuda")
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0   # tt_debug_set_fused
tt.tt_debug_set_fused(mode)
if len(sys.argv) > 4:
    tt.tt_debug_set_variant(int(sys.argv[4]))   # forced tile configuration (tt_launch_tpl.cuh)
for name, fn in (("left", lambda: tt.tt_interface_left(phiL, A, x, workspace=wi)),
                 ("right", lambda: tt.tt_interface_right(phiR, A, x, workspace=wi))):
    fn()
    torch.cuda.synchronize()
    tt.tt_trace_enable(1000)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
    tt.tt_trace_disable()
    agg = {}
    for rec in recs:
        d = agg.setdefault(rec["stage"], [0.0, 0.0, rec["M"], rec["N"], rec["K"], rec["tile"]])
        d[0] += rec["ms"] / 5
        d[1] += 2.0 * rec["M"] * rec["N"] * rec["K"] / 5
    tot = sum(v[0] for v in agg.values())
    print(name, f"total {tot:.3f} ms", "  ".join(
        f"{k}: {v[0]:.3f} ms {v[1] / v[0] / 1e9:.1f} TF (M={v[2]} N={v[3]} K={v[4]} tile={v[5]})"
        for k, v in agg.items()), flush=True)
