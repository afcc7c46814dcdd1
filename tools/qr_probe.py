"""Traced time of one cluster Householder QR (tt_qr.cuh) per unfolding shape."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402

for m, c in [(1024, 256), (1024, 64), (256, 256), (256, 64), (64, 16)]:
    rng = np.random.default_rng(1)
    n0 = 4
    r0 = m // n0
    x = [rng.standard_normal((1, n0, r0)), rng.standard_normal((r0, n0, c)), rng.standard_normal((c, n0, 1))]
    xg = [torch.from_numpy(t).cuda() for t in x]
    tt.tt_orthonormalise(xg, tt.TT_SWEEP_LEFT)
    torch.cuda.synchronize()
    tt.tt_trace_enable(100)
    tt.tt_orthonormalise(xg, tt.TT_SWEEP_LEFT)
    torch.cuda.synchronize()
    recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
    tt.tt_trace_disable()
    qr = [r for r in recs if r["tile"] == -3]
    print(f"{m} x {c}: " + ", ".join(f"QR {r['M']}x{r['N']} {r['ms'] * 1e3:.1f} us" for r in qr), flush=True)
