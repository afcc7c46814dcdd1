"""Time the cooperative Jacobi eigensolver (tt_debug_sym_eigen) on random SPD Gram matrices."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402

for n in [int(a) for a in (sys.argv[1:] or ["64", "128", "256", "512"])]:
    g = torch.Generator(device="cuda").manual_seed(n)
    M = torch.randn(4 * n, n, dtype=torch.float64, device="cuda", generator=g)
    G = M.T @ M
    tt.tt_debug_sym_eigen(G)
    torch.cuda.synchronize()
    t = time.perf_counter()
    lam, V = tt.tt_debug_sym_eigen(G)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) * 1e3
    err = (G @ V - V * lam).abs().max().item() / lam.abs().max().item()
    print(f"n={n}: {dt:.2f} ms  residual {err:.1e}", flush=True)
