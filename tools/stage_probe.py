"""Per-stage GEMM timing at config-5 interior-core shapes under the benchmark hooks
(variant x {normal, no-stores, no-loads, neither}); prints TF/s per stage."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402


def run(variant, flags, a=256, b=256, al=36, be=36, n=4, K=32, reps=3):
    tt.tt_debug_set_variant(variant)
    tt.tt_debug_set_flags(flags)
    g = torch.Generator(device="cuda").manual_seed(0)
    r = lambda *s: torch.randn(*s, dtype=torch.float64, device="cuda", generator=g)
    phiL, A, phiR, X = r(a, al, a), r(al, n, n, be), r(b, be, b), r(a, n, K, b)
    Y = torch.empty_like(X)
    ws = torch.empty(tt.tt_local_matvec_workspace_size(a, n, b, al, be, K), dtype=torch.uint8,
                     device="cuda")
    tt.tt_local_matvec_batched(phiL, A, phiR, X, Y, workspace=ws)
    torch.cuda.synchronize()
    tt.tt_trace_enable(1000)
    for _ in range(reps):
        tt.tt_local_matvec_batched(phiL, A, phiR, X, Y, workspace=ws)
    torch.cuda.synchronize()
    recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
    tt.tt_trace_disable()
    tt.tt_debug_set_flags(0)
    out = {}
    for rec in recs:
        if rec["stage"].startswith("mv_"):
            d = out.setdefault(rec["stage"], [0.0, 0.0])
            d[0] += rec["ms"]
            d[1] += 2.0 * rec["M"] * rec["N"] * rec["K"]
    return {k: (v[0] / reps, v[1] / v[0] / 1e9) for k, v in out.items()}


if __name__ == "__main__":
    for variant in [int(v) for v in (sys.argv[1:] or ['1', '2'])]:
        sets = ((0, "normal"), (16, "no-L2-hints"), (32, "no-evict-first"), (64, "no-evict-last"),
                (128, "2d-boxes"), (1, "no-stores"), (2, "no-loads"), (3, "compute-only"))
        if os.environ.get("PROBE_QUICK"):
            sets = ((0, "normal"), (3, "compute-only"))
        if os.environ.get("PROBE_UNITS"):
            sets = ((0, "fast-units"), (524288, "div-units"), (0, "fast-units"), (524288, "div-units"))
        if os.environ.get("PROBE_CTAB"):
            sets = ((0, "col-table"), (262144, "col-map"), (0, "col-table"), (262144, "col-map"))
        if os.environ.get("PROBE_QUAD"):
            sets = ((0, "quad-stores"), (131072, "pair-stores"), (1, "no-stores"), (0, "quad-stores"))
        if os.environ.get("PROBE_SKEW"):
            sets = ((0, "skew0"), (16384, "skew1"), (32768, "skew2"), (0, "skew0"))
        if os.environ.get("PROBE_BRES"):
            sets = ((0, "ring-B"), (33554432, "resident-B"), (0, "ring-B"), (33554432, "resident-B"))
        if os.environ.get("PROBE_RASTER"):
            sets = ((0, "n-fastest"), (512, "group-m-8"), (1024, "m-fastest"))
        for flags, name in sets:
            res = run(variant, flags)
            print(f"variant {variant} {name:13s} " + "  ".join(
                f"{k}: {ms:.3f} ms {tf:.2f} TF" for k, (ms, tf) in sorted(res.items())), flush=True)
