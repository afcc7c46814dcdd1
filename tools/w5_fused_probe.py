"""Config-5 W5 sweep (tt_sweep_als, K = 32) with the three-stage matvec and with the fused
S1 -> S2 kernel (tt_debug_set_fused): CUDA-event time of the whole sweep, best of `reps`.
Usage: python tools/w5_fused_probe.py [--modes=-1,2] [--reps 4]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--modes", default="-1,2")
ap.add_argument("--reps", type=int, default=4)
args = ap.parse_args()
inp = ttgen.make_inputs(5)
xs = [torch.from_numpy(c).cuda() for c in inp.x]
As = [torch.from_numpy(c).cuda() for c in inp.A]
Xs = [torch.from_numpy(c).cuda() for c in inp.X]
ref = None
for mode in [int(m) for m in args.modes.split(",")]:
    tt.tt_debug_set_fused(mode)
    Yf, _, pl, pr = tt.tt_sweep_als(xs, As, Xs)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(args.reps):
        ev0.record()
        tt.tt_sweep_als(xs, As, Xs, Yf, None, pl, pr)
        ev1.record()
        torch.cuda.synchronize()
        best = min(best, ev0.elapsed_time(ev1))
    if ref is None:
        ref = [y.clone() for y in Yf]
        err = 0.0
    else:
        err = max(float((y - r).norm() / r.norm()) for y, r in zip(Yf, ref))
    print(f"mode {mode:2d}: W5 sweep {best:.3f} ms | max rel diff of Y vs first mode {err:.2e}", flush=True)
tt.tt_debug_set_fused(0)
