"""Per-launch trace of one config-5 W5 sweep (sequential-equivalent timings are not
available for the overlapped interface chains; matvec stages are on the main stream).
Prints the launches that lose the most time against the 37 TF/s DMMA peak."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

inp = ttgen.make_inputs(5)
xs = [torch.from_numpy(c).cuda() for c in inp.x]
As = [torch.from_numpy(c).cuda() for c in inp.A]
Xs = [torch.from_numpy(c).cuda() for c in inp.X]
Yf, _, pl, pr = tt.tt_sweep_als(xs, As, Xs)
torch.cuda.synchronize()
tt.tt_trace_enable(4000)
tt.tt_sweep_als(xs, As, Xs, Yf, None, pl, pr)
torch.cuda.synchronize()
recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
tt.tt_trace_disable()
P = 37.0e12
rows = []
for r in recs:
    if r["stage"].startswith("mv_"):
        f = 2.0 * r["M"] * r["N"] * r["K"]
        lost = r["ms"] - f / P * 1e3
        rows.append((lost, r["stage"], r["M"], r["N"], r["K"], r["tile"], r["ms"], f / r["ms"] / 1e9))
rows.sort(reverse=True)
print("lost_ms stage M N K tile ms TF")
for row in rows[:24]:
    print(f"{row[0]:.3f} {row[1]} {row[2]} {row[3]} {row[4]} {row[5]} {row[6]:.3f} {row[7]:.2f}")
print("total matvec lost ms:", sum(r[0] for r in rows))
