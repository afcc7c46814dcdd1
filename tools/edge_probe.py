"""Matvec stage times at the config-5 boundary-adjacent cores (k = 3: a = 64, b = 256 and
k = 8: a = 256, b = 64; alpha = beta = 36, N = 4, K = 32) under forced GEMM variants."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from stage_probe import run  # noqa: E402

for variant in [int(v) for v in (sys.argv[1:] or ["-1"])]:
    for a, b in ((64, 256), (256, 64)):
        res = run(variant, 0, a=a, b=b)
        print(f"variant {variant} a={a} b={b} " + "  ".join(
            f"{k}: {ms:.3f} ms {tf:.2f} TF" for k, (ms, tf) in sorted(res.items())), flush=True)
