"""cuBLAS DGEMM reference peak via torch.matmul float64 (SURVEY.md §8(d) P64 recipe).

Not part of the product path: torch is used here only to time the vendor library as a
roofline denominator.  Prints one JSON line.
"""
import json
import time

import torch


def main(n: int = 8192) -> None:
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    flops = 2.0 * n ** 3
    best = 1e30
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    # sustained: back to back for ~4 s
    t0 = time.time()
    cnt = 0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.time() - t0 < 4.0:
        for _ in range(10):
            torch.matmul(a, b, out=c)
        cnt += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sustained_ms = e0.elapsed_time(e1) / cnt
    print(json.dumps({"kind": "cublas_dgemm", "n": n, "best_ms": best,
                      "tflops_burst": flops / best / 1e9,
                      "tflops_sustained": flops / sustained_ms / 1e9}))


if __name__ == "__main__":
    main()
