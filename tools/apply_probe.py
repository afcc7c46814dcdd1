"""Time tt_operator_apply on config-5 cores (HBM-bound): GB/s per core and in total."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

cfg = ttgen.CONFIGS[5]
g = torch.Generator(device="cuda").manual_seed(0)
xs = [torch.randn(cfg.r[k], cfg.N, cfg.r[k + 1], dtype=torch.float64, device="cuda", generator=g)
      for k in range(cfg.d)]
As = [torch.randn(cfg.R[k], cfg.N, cfg.N, cfg.R[k + 1], dtype=torch.float64, device="cuda", generator=g)
      for k in range(cfg.d)]
zs = tt.tt_operator_apply(xs, As)
torch.cuda.synchronize()
tt.tt_trace_enable(1000)
for _ in range(3):
    tt.tt_operator_apply(xs, As, zs)
torch.cuda.synchronize()
recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
tt.tt_trace_disable()
tot_ms = sum(r["ms"] for r in recs) / 3
tot_b = sum(8 * (x.numel() + A.numel() + z.numel()) for x, A, z in zip(xs, As, zs))
print(f"apply: {tot_ms:.3f} ms  {tot_b / tot_ms / 1e6:.0f} GB/s")
for k in range(cfg.d):
    ms = sum(r["ms"] for r in recs[k::cfg.d]) / 3
    b = 8 * (xs[k].numel() + As[k].numel() + zs[k].numel())
    print(f"  core {k}: {ms:.4f} ms {b / ms / 1e6:.0f} GB/s")
