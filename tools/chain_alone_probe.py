"""Graph-replay time of the interface chains alone (left, right, both) and of W34, configs 3/4:
how much of W34 is the two chains, and how well the two concurrent chains overlap."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402


def graph_time(fn, reps=30):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn(s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2] * 1e3


for idx in [int(a) for a in (sys.argv[1:] or ["3", "4"])]:
    inp = ttgen.make_inputs(idx)
    x = [torch.from_numpy(c).cuda() for c in inp.x]
    A = [torch.from_numpy(c).cuda() for c in inp.A]
    tr = tt._Train(x, A)
    pl, pr = tt.alloc_interfaces(x, A), tt.alloc_interfaces(x, A)
    y = [torch.empty_like(c) for c in x]
    ws = torch.empty(max(tt.tt_sweep_w34_workspace_size(tr), tt.tt_sweep_workspace_size(tr)),
                     dtype=torch.uint8, device="cuda")
    res = {}
    for name, dirs in [("left", tt.TT_SWEEP_LEFT), ("right", tt.TT_SWEEP_RIGHT), ("both", tt.TT_SWEEP_BOTH)]:
        res[name] = graph_time(lambda s, d=dirs: tt.tt_sweep_interfaces(x, A, pl, pr, d, workspace=ws, stream=s))
    res["w34"] = graph_time(lambda s: tt.tt_sweep_w34(x, A, pl, pr, y, workspace=ws, stream=s))
    print(f"config {idx}: " + "  ".join(f"{k} {v:.1f} us" for k, v in res.items()), flush=True)
