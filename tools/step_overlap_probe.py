"""Bench step (config 5: W5 sweep + apply): apply after the sweep on the same stream vs the
apply on a forked low- / high-priority stream concurrently with the sweep (it only reads x, A)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

inp = ttgen.make_inputs(5)
dev = torch.device("cuda")
x = [torch.from_numpy(c).to(dev) for c in inp.x]
A = [torch.from_numpy(c).to(dev) for c in inp.A]
X = [torch.from_numpy(c).to(dev) for c in inp.X]
Y = [torch.empty_like(t) for t in X]
pl, pr = tt.alloc_interfaces(x, A), tt.alloc_interfaces(x, A)
z = tt.tt_operator_apply(x, A)
ws = torch.empty(tt.tt_sweep_als_workspace_size(tt._Train(x, A), 32), dtype=torch.uint8, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
main = torch.cuda.Stream()
lo, hi = torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-1)
sweep = tt.prepare(tt.tt_sweep_als, x, A, X, Y, None, pl, pr, workspace=ws, stream=main)
apply_ = tt.prepare(tt.tt_operator_apply, x, A, z, stream=main)


def step(mode):
    if mode == "serial":
        sweep(main)
        apply_(main)
        return
    side = lo if mode == "lowprio" else hi
    side.wait_stream(main)
    apply_(side)
    sweep(main)
    main.wait_stream(side)


torch.cuda.synchronize()
for rep in range(2):
    for mode in ("serial", "lowprio", "hiprio"):
        ts = []
        for it in range(6):
            with torch.cuda.stream(main):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(main)
                step(mode)
                e1.record(main)
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(e0.elapsed_time(e1))
        print(f"{mode:8s}: {sorted(ts)[len(ts) // 2]:.2f} ms (min {min(ts):.2f})", flush=True)
