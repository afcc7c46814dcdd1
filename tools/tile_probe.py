"""Latency tile-policy probe: every stage GEMM of the left interface update and of the
single-vector local matvec at the config-3/4 core shapes, under each forced tile configuration
(tt_debug_set_variant 10..22, + 100 x forced split-K), timed by the library's event tracer.
Prints, per stage shape, the default's time and the best forced configuration."""
import collections
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402

N = 4
SHAPES = [(16, 64, 16, 16), (64, 64, 16, 16), (64, 16, 16, 16),
          (16, 64, 25, 25), (64, 128, 25, 25), (128, 128, 25, 25), (128, 64, 25, 25),
          (64, 16, 25, 25)]
CFGS = list(range(10, 23))
KS = [0, 1, 2, 4, 8]
REPS = 5


def run_shape(a, b, al, be, variant):
    g = torch.Generator(device="cuda").manual_seed(0)
    r = lambda *s: torch.randn(*s, dtype=torch.float64, device="cuda", generator=g)
    phiL, A, phiR, x = r(a, al, a), r(al, N, N, be), r(b, be, b), r(a, N, b)
    out = torch.empty(b, be, b, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    wi = torch.empty(tt.tt_interface_workspace_size(a, N, b, al, be), dtype=torch.uint8, device="cuda")
    wm = torch.empty(tt.tt_local_matvec_workspace_size(a, N, b, al, be, 1), dtype=torch.uint8,
                     device="cuda")
    tt.tt_debug_set_variant(variant)
    try:
        tt.tt_interface_left(phiL, A, x, out, workspace=wi)
        tt.tt_local_matvec(phiL, A, phiR, x, y, workspace=wm)
        torch.cuda.synchronize()
        tt.tt_trace_enable(10000)
        for _ in range(REPS):
            tt.tt_interface_left(phiL, A, x, out, workspace=wi)
            tt.tt_local_matvec(phiL, A, phiR, x, y, workspace=wm)
        torch.cuda.synchronize()
        recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
    finally:
        tt.tt_trace_disable()
        tt.tt_debug_set_variant(-1)
    per = collections.defaultdict(list)
    for rec in recs:
        if rec["stage"] in ("perm", "set"):
            continue
        per[(rec["stage"], rec["M"], rec["N"], rec["K"])].append((rec["ms"] * 1e3, rec["tile"]))
    return {k: (statistics.median(t for t, _ in v), v[0][1]) for k, v in per.items()}


results = {}
for shp in SHAPES:
    base = run_shape(*shp, -1)
    best = {k: (v[0], "default", v[1]) for k, v in base.items()}
    for c in CFGS:
        for ks in KS:
            res = run_shape(*shp, c + 100 * ks)
            for k, (us, tile) in res.items():
                if k in best and us < best[k][0]:
                    best[k] = (us, f"cfg{c} ks{ks}", tile)
    for k in base:
        print(f"{shp} {k[0]:6s} M={k[1]:6d} N={k[2]:5d} K={k[3]:5d}  default {base[k][0]:7.2f} us "
              f"(tile {base[k][1]})  best {best[k][0]:7.2f} us {best[k][1]} (tile {best[k][2]})",
              flush=True)
        results[f"{shp} {k}"] = {"default_us": base[k][0], "best_us": best[k][0], "best": best[k][1]}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(results, open("gpurun_out/tile_probe.json", "w"), indent=1)
