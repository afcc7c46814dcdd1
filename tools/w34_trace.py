"""Per-launch trace of ONE tt_sweep_w34 call (stream version): per stage tag the launches,
summed traced ms and TFLOP/s, and the wall time of the call."""
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
tt.tt_set_graph_cache(False)
for _ in range(3):
    tt.tt_sweep_w34(x, A)
torch.cuda.synchronize()
tt.tt_trace_enable(4000)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
tt.tt_sweep_w34(x, A)
e1.record()
torch.cuda.synchronize()
recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
tt.tt_trace_disable()
print(f"W34 config {idx}: {e0.elapsed_time(e1):.3f} ms wall (eager, traced), {len(recs)} launches")
for r in recs:
    f = 2.0 * r["M"] * r["N"] * r["K"] if r["N"] else 0.0
    print(f"  {r['stage']:6s} tile {r['tile']:7d}  M {r['M']:7d} N {r['N']:6d} K {r['K']:6d}  "
          f"{r['ms'] * 1e3:8.1f} us  {f / r['ms'] / 1e9 if r['ms'] else 0:6.2f} TF/s  {f / 1e9:7.3f} GF")
