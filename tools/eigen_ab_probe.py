"""A/B of the block Jacobi eigensolver kernels (tt_debug_sym_eigen): default (cross-pair inner
sweeps, two-rsqrt rotations, DMMA updates, blocks of 16), debug bit 2 (the same with blocks of
32), debug bit 16 (the first kernel: full inner sweeps, scalar updates), bit 8 (element-wise).  Random SPD Gram matrices and a graded one."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402

for n in [int(a) for a in (sys.argv[1:] or ["8", "16", "32", "64", "128", "256", "512", "1024"])]:
    g = torch.Generator(device="cuda").manual_seed(n)
    M = torch.randn(4 * n, n, dtype=torch.float64, device="cuda", generator=g)
    Gs = {"random": M.T @ M}
    Q = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g))[0]
    sig = torch.logspace(0, -12, n, dtype=torch.float64, device="cuda")
    Gs["graded"] = (Q * sig) @ Q.T
    for name, G in Gs.items():
        for flags, label in [(0, "v2 BS=16"), (1 << 2, "v2 BS=32"), (1 << 16, "v1"),
                             (1 << 8, "element-wise")]:
            if flags == 1 << 8 and n > 128:
                continue
            tt.tt_debug_set_flags(flags)
            tt.tt_debug_sym_eigen(G)
            torch.cuda.synchronize()
            t = time.perf_counter()
            lam, V = tt.tt_debug_sym_eigen(G)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t) * 1e3
            err = (G @ V - V * lam).abs().max().item() / lam.abs().max().item()
            orth = (V.T @ V - torch.eye(n, dtype=torch.float64, device="cuda")).abs().max().item()
            print(f"n={n} {name:7s} {label:14s}: {dt:7.2f} ms  residual {err:.1e}  orth {orth:.1e}",
                  flush=True)
tt.tt_debug_set_flags(0)
