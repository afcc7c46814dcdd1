"""W34 DAG (configs 3, 4) CUDA-graph time under the latency-model knobs in the environment
(TT_LAT_FLOPS, TT_LAT_UNIT_US, TT_LAT_MASK, TT_LAT_SPLIT_US, TT_LAT_OCC, TT_PDL_FLOPS); one line per process."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

tt.tt_debug_set_flags(int(os.environ.get("TT_FLAGS", "0")))   # debug bits (header)
out = []
for idx in (3, 4):
    inp = ttgen.make_inputs(idx)
    x = [torch.from_numpy(c).cuda() for c in inp.x]
    A = [torch.from_numpy(c).cuda() for c in inp.A]
    pl, pr = tt.alloc_interfaces(x, A), tt.alloc_interfaces(x, A)
    y = [torch.empty_like(c) for c in x]
    ws = torch.empty(tt.tt_sweep_w34_workspace_size(tt._Train(x, A)), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    f = lambda: tt.tt_sweep_w34(x, A, pl, pr, y, workspace=ws, stream=s)
    f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            f()
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out.append(f"c{idx} {statistics.median(ts):.3f} ms")
knobs = {k: v for k, v in os.environ.items() if k.startswith(("TT_LAT", "TT_PDL", "TT_FLAGS"))}
print(knobs, " ".join(out), flush=True)
