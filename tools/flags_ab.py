"""A/B the debug flags (tt_debug_set_flags) on the config-5 W5 sweep + apply step:
interleaved repetitions, CUDA-event timed, L2 flushed between steps.
usage: python tools/flags_ab.py FLAGS_A FLAGS_B [reps]   (a token "vN" selects GEMM variant N
instead of debug flags)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

fa, fb = sys.argv[1], sys.argv[2]


def apply(tok):
    if tok.startswith("v"):
        tt.tt_debug_set_flags(0)
        tt.tt_debug_set_variant(int(tok[1:]))
    else:
        tt.tt_debug_set_variant(-1)
        tt.tt_debug_set_flags(int(tok))

reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
inp = ttgen.make_inputs(5)
xs = [torch.from_numpy(c).cuda() for c in inp.x]
As = [torch.from_numpy(c).cuda() for c in inp.A]
Xs = [torch.from_numpy(c).cuda() for c in inp.X]
Yf, _, pl, pr = tt.tt_sweep_als(xs, As, Xs)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
res = {fa: [], fb: []}
for rep in range(reps + 1):
    for f in (fa, fb):
        apply(f)
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tt.tt_sweep_als(xs, As, Xs, Yf, None, pl, pr)
        e1.record()
        torch.cuda.synchronize()
        if rep:
            res[f].append(e0.elapsed_time(e1))
tt.tt_debug_set_flags(0)
tt.tt_debug_set_variant(-1)
for f in (fa, fb):
    v = sorted(res[f])
    print(f"flags {f}: median {v[len(v) // 2]:.3f} ms  min {v[0]:.3f}  all {[round(x, 2) for x in res[f]]}")
