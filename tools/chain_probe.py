"""Left interface chain of config 3 / 4 alone: CUDA-graph replay time and launch count, so the
per-launch gap of a dependent kernel chain can be read against the ncu launch list of the same
chain (`python tools/chain_probe.py <cfg> once` runs it exactly once for ncu)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 3
once = len(sys.argv) > 2 and sys.argv[2] == "once"
inp = ttgen.make_inputs(idx)
x = [torch.from_numpy(c).cuda() for c in inp.x]
A = [torch.from_numpy(c).cuda() for c in inp.A]
pl = tt.alloc_interfaces(x, A)
tr = tt._Train(x, A)
ws = torch.empty(tt.tt_sweep_workspace_size(tr), dtype=torch.uint8, device="cuda")


def left(s):
    tt.tt_sweep_interfaces(x, A, pl, None, directions=tt.TT_SWEEP_LEFT, workspace=ws, stream=s)


s = torch.cuda.Stream()
left(s)
torch.cuda.synchronize()
if once:
    left(s)
    torch.cuda.synchronize()
    sys.exit(0)
launches = tt.tt_last_launch_count()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        left(s)
torch.cuda.synchronize()
ts = []
for _ in range(50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"config {idx} left chain: {launches} launches, graph {statistics.median(ts)*1e3:.1f} us "
      f"({statistics.median(ts)*1e3/launches:.2f} us per launch)")
