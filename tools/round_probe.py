"""tt_round of the config-5 vector train, repeated, under debug flags (0 / no-PDL / no latency
tiles): host wall time per call and whether repeated calls give bit-identical cores."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

inp = ttgen.make_inputs(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
xs = [torch.from_numpy(c).cuda() for c in inp.x]
for flags in [int(f) for f in (sys.argv[2:] or ["0", "4096", "8192", "0"])]:
    tt.tt_debug_set_flags(flags)
    ts, outs = [], []
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = tt.tt_round(xs, 1e-4)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
        outs.append([c.clone() for c in out])
    same = all(torch.equal(a, b) for o in outs[1:] for a, b in zip(o, outs[0]))
    print(f"flags {flags}: ms {[round(t, 1) for t in ts]} ranks {[c.shape[2] for c in outs[0]]} "
          f"identical {same}", flush=True)
tt.tt_debug_set_flags(0)
