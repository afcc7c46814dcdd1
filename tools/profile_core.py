"""Profiling driver: one batched local matvec (and optionally one interface update) at the
config-5 interior-core shapes (a=b=256, alpha=beta=36, N=4, K=32), repeated `reps` times.
Launch order per matvec: perm, S1, S2, S3 (so `ncu -k regex:dmma_gemm -s 6 -c 3` captures
the three GEMM stages of the third repetition)."""
import argparse
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--what", default="matvec", choices=["matvec", "left", "right"])
    ap.add_argument("--a", type=int, default=256)
    ap.add_argument("--b", type=int, default=256)
    ap.add_argument("--al", type=int, default=36)
    ap.add_argument("--be", type=int, default=36)
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--K", type=int, default=32)
    args = ap.parse_args()
    a, b, al, be, n, K = args.a, args.b, args.al, args.be, args.n, args.K
    g = torch.Generator(device="cuda").manual_seed(0)
    r = lambda *s: torch.randn(*s, dtype=torch.float64, device="cuda", generator=g)
    phiL, A, phiR = r(a, al, a), r(al, n, n, be), r(b, be, b)
    X = r(a, n, K, b)
    x = r(a, n, b)
    Y = torch.empty_like(X)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(args.reps):
        ev0.record()
        if args.what == "matvec":
            tt.tt_local_matvec_batched(phiL, A, phiR, X, Y)
        elif args.what == "left":
            tt.tt_interface_left(phiL, A, x)
        else:
            tt.tt_interface_right(phiR, A, x)
        ev1.record()
        torch.cuda.synchronize()
        print(f"rep {i}: {ev0.elapsed_time(ev1):.3f} ms", flush=True)


if __name__ == "__main__":
    main()
