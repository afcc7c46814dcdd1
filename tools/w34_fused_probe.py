"""tt_sweep_w34 (graph replay) at config `idx` with the stage GEMMs and with the fused S1 -> S2
kernel forced into every eligible interface update (tt_debug_set_fused): time and launches.
Usage: python tools/w34_fused_probe.py [idx] [--modes=-1,2]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 3
modes = [-1, 2]
for a in sys.argv[2:]:
    if a.startswith("--modes="):
        modes = [int(m) for m in a.split("=")[1].split(",")]
inp = ttgen.make_inputs(idx)
xs = [torch.from_numpy(c).cuda() for c in inp.x]
As = [torch.from_numpy(c).cuda() for c in inp.A]
pl, pr = tt.alloc_interfaces(xs, As), tt.alloc_interfaces(xs, As)
ys = [torch.empty_like(t) for t in xs]
w = torch.empty(tt.tt_sweep_w34_workspace_size(tt._Train(xs, As)), dtype=torch.uint8, device="cuda")
ref = None
for mode in modes:
    tt.tt_debug_set_fused(mode)
    stream = torch.cuda.current_stream()
    for _ in range(3):
        tt.tt_sweep_w34(xs, As, pl, pr, ys, workspace=w)
    n = tt.tt_last_launch_count()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(stream)
    with torch.cuda.stream(cap):
        with torch.cuda.graph(g, stream=cap):
            tt.tt_sweep_w34(xs, As, pl, pr, ys, workspace=w, stream=cap)
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    if ref is None:
        ref = [y.clone() for y in ys]
        err = 0.0
    else:
        err = max(float((y - r).norm() / r.norm()) for y, r in zip(ys, ref))
    print(f"config {idx} mode {mode:2d}: W34 graph median {ts[len(ts) // 2] * 1e3:.1f} us best {ts[0] * 1e3:.1f} us, "
          f"{n} launches, max rel diff {err:.1e}", flush=True)
    del g
tt.tt_debug_set_fused(0)
