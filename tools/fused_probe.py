"""Fused S1 -> S2 matvec kernel (csrc/tt_fused12.cuh) against the three-stage path at the
config-5 interior-core shape (a = b = 256, al = be = 36, N = 4, K = 32): per-stage times from
the tracer, whole-matvec time from CUDA events, max difference of the results.
Usage: python tools/fused_probe.py [--modes -1,1,2,3] [--reps 5] [--a .. --b .. --al .. --be .. --K ..]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--modes", default="-1,1,2,3")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--a", type=int, default=256)
    ap.add_argument("--b", type=int, default=256)
    ap.add_argument("--al", type=int, default=36)
    ap.add_argument("--be", type=int, default=36)
    ap.add_argument("--K", type=int, default=32)
    args = ap.parse_args()
    a, b, al, be, K, n = args.a, args.b, args.al, args.be, args.K, 4
    g = torch.Generator(device="cuda").manual_seed(0)
    r = lambda *s: torch.randn(*s, dtype=torch.float64, device="cuda", generator=g)
    phiL, A, phiR, X = r(a, al, a), r(al, n, n, be), r(b, be, b), r(a, n, K, b)
    flops = 2.0 * n * K * (a * a * al * b + a * b * b * be) + 2.0 * a * b * al * be * n * n * K
    ref = None
    tt.tt_set_graph_cache(False)
    for mode in [int(m) for m in args.modes.split(",")]:
        tt.tt_debug_set_fused(mode)
        Y = torch.empty_like(X)
        tt.tt_local_matvec_batched(phiL, A, phiR, X, Y)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(args.reps):
            ev0.record()
            tt.tt_local_matvec_batched(phiL, A, phiR, X, Y)
            ev1.record()
            torch.cuda.synchronize()
            best = min(best, ev0.elapsed_time(ev1))
        tt.tt_trace_enable(64)
        tt.tt_local_matvec_batched(phiL, A, phiR, X, Y)
        torch.cuda.synchronize()
        recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
        tt.tt_trace_disable()
        st = " ".join(f"{q['stage']}[{q['tile']}]={q['ms']:.3f}ms/{2.0 * q['M'] * q['N'] * q['K'] / q['ms'] / 1e9:.2f}TF"
                      for q in recs if q["stage"].startswith("mv_"))
        if ref is None:
            ref = Y.clone()
            err = 0.0
        else:
            err = float((Y - ref).norm() / ref.norm())
        print(f"mode {mode:2d}: matvec {best:.3f} ms {flops / best / 1e9:.2f} TF/s | {st} | rel diff vs first {err:.2e}",
              flush=True)
    tt.tt_debug_set_fused(0)


if __name__ == "__main__":
    main()
