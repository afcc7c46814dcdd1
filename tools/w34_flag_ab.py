"""W34 graph-replay time per config for a list of debug flag values (A/B in one process)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

flags = [int(f, 0) for f in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0]
for idx in (2, 3, 4):
    inp = ttgen.make_inputs(idx)
    x = [torch.from_numpy(c).cuda() for c in inp.x]
    A = [torch.from_numpy(c).cuda() for c in inp.A]
    pl, pr = tt.alloc_interfaces(x, A), tt.alloc_interfaces(x, A)
    y = [torch.empty_like(c) for c in x]
    ws = torch.empty(tt.tt_sweep_w34_workspace_size(tt._Train(x, A)), dtype=torch.uint8, device="cuda")
    res = []
    for rep in range(2):
        for f in flags:
            tt.tt_debug_set_flags(f)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                tt.tt_sweep_w34(x, A, pl, pr, y, workspace=ws, stream=s)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    tt.tt_sweep_w34(x, A, pl, pr, y, workspace=ws, stream=s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ts = []
            for _ in range(30):
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res.append((f, sorted(ts)[15] * 1e3))
    tt.tt_debug_set_flags(0)
    print(f"config {idx}: " + "  ".join(f"{f:#x}: {t:.1f} us" for f, t in res), flush=True)
