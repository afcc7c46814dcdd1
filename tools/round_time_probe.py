"""Host wall time of tt_round / tt_orthonormalise on the config-5 vector train: QR path vs the
Gram route (debug bit 29); round at 1e-10 and 0 takes the accurate truncation (QR + Jacobi SVD),
and at 1e-4 with debug bit 24 forced."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

inp = ttgen.make_inputs(5)
x = [torch.from_numpy(c).cuda() for c in inp.x]
for flags, name in [(0, "QR"), (1 << 29, "Gram"), (1 << 24, "Acc")]:
    tt.tt_debug_set_flags(flags)
    for fn, label in [(lambda: tt.tt_orthonormalise(x, tt.TT_SWEEP_LEFT), "orthonormalise left"),
                      (lambda: tt.tt_orthonormalise(x, tt.TT_SWEEP_RIGHT), "orthonormalise right"),
                      (lambda: tt.tt_round(x, 1e-4), "round 1e-4"),
                      (lambda: tt.tt_round(x, 1e-10), "round 1e-10"),
                      (lambda: tt.tt_round(x, 0.0), "round 0")]:
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            out = fn()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"{name:5s} {label:22s} {min(ts):8.2f} ms  ranks {[int(c.shape[2]) for c in out][:6]}",
              flush=True)
tt.tt_debug_set_flags(0)
