"""Per-launch trace of the config-4 W34 sweep (all interfaces + one matvec per core)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
inp = ttgen.make_inputs(idx)
x = [torch.from_numpy(c).cuda() for c in inp.x]
A = [torch.from_numpy(c).cuda() for c in inp.A]
pl, pr = tt.tt_sweep_interfaces(x, A)
ys = [tt.tt_local_matvec(pl[k], A[k], pr[k + 1], x[k]) for k in range(len(x))]
torch.cuda.synchronize()
tt.tt_trace_enable(4000)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
tt.tt_sweep_interfaces(x, A, pl, pr)
for k in range(len(x)):
    tt.tt_local_matvec(pl[k], A[k], pr[k + 1], x[k], ys[k])
e1.record()
torch.cuda.synchronize()
recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
tt.tt_trace_disable()
print(f"W34 config {idx}: {e0.elapsed_time(e1):.3f} ms, traced {sum(r['ms'] for r in recs):.3f} ms, {len(recs)} launches")
agg = {}
for r in recs:
    a = agg.setdefault(r["stage"], [0, 0.0, 0.0])
    a[0] += 1
    a[1] += r["ms"]
    a[2] += 2.0 * r["M"] * r["N"] * r["K"] if r["N"] else 0
for k, (n, ms, f) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {k:6s} {n:3d} launches {ms:.3f} ms {f / ms / 1e9 if ms else 0:.2f} TF")
worst = sorted(recs, key=lambda r: -r["ms"])[:12]
for r in worst:
    print("   ", r)
