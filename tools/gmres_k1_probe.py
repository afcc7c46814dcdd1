"""K = 1 GMRES(m) latency at config-3/4 interior shapes: fused cluster orthogonalisation vs the
separate kernels (debug flag 1 << 26), CUDA-graph replay, per Arnoldi step."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402


def timeit(fn, reps=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


for (a, al, name) in [(64, 16, "config3"), (128, 25, "config4")]:
    N, m = 4, 10
    rng = np.random.default_rng(1)
    g = lambda x: torch.from_numpy(x).cuda()
    phL = g(rng.standard_normal((a, al, a)) / a)
    phR = g(rng.standard_normal((a, al, a)) / a)
    A = g(rng.standard_normal((al, N, N, al)) / np.sqrt(al * N))
    F = g(rng.standard_normal((a, N, 1, a)))
    X = torch.zeros_like(F)
    rel = torch.zeros(1, dtype=torch.float64, device="cuda")
    its = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(tt.tt_local_gmres_workspace_size(a, N, a, al, al, 1, m), dtype=torch.uint8, device="cuda")
    for flags in (0, 1 << 26):
        tt.tt_debug_set_flags(flags)
        s = torch.cuda.Stream()
        run = lambda: tt.tt_local_gmres(phL, A, phR, F, X, m=m, cycles=1, tol=0.0, rel_res=rel,
                                        iters=its, workspace=ws, stream=s)
        with torch.cuda.stream(s):
            run()
            torch.cuda.synchronize()
            n = tt.tt_last_launch_count()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                run()
        t = timeit(gr.replay)
        tmv = None
        print(f"{name} a={a} alpha={al} m={m} flags={flags:#x}: {t * 1e3:.1f} us per GMRES({m}) cycle, "
              f"{t * 1e3 / m:.1f} us per Arnoldi step, {n} launches, its={int(its.item())}, rel={rel.item():.2e}",
              flush=True)
    tt.tt_debug_set_flags(0)

# per-launch trace of one eager K = 1 cycle (config-3 shape), fused orthogonalisation
a, al, N, m = 64, 16, 4, 10
rng = np.random.default_rng(1)
g = lambda x: torch.from_numpy(x).cuda()
phL = g(rng.standard_normal((a, al, a)) / a)
phR = g(rng.standard_normal((a, al, a)) / a)
A = g(rng.standard_normal((al, N, N, al)) / np.sqrt(al * N))
F = g(rng.standard_normal((a, N, 1, a)))
for flags in (0, 1 << 26):
    tt.tt_debug_set_flags(flags)
    tt.tt_local_gmres(phL, A, phR, F, m=m, cycles=1, tol=0.0)
    torch.cuda.synchronize()
    tt.tt_trace_enable(2000)
    tt.tt_local_gmres(phL, A, phR, F, m=m, cycles=1, tol=0.0)
    torch.cuda.synchronize()
    recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
    tt.tt_trace_disable()
    agg = {}
    for r in recs:
        key = (r["stage"], r["tile"], r["M"], r["N"], r["K"])
        a_ = agg.setdefault(key, [0, 0.0])
        a_[0] += 1
        a_[1] += r["ms"]
    print(f"flags={flags:#x}: traced {len(recs)} launches, {sum(r['ms'] for r in recs) * 1e3:.1f} us total")
    for key, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"   {key}: {n} x {ms / n * 1e3:.2f} us")
tt.tt_debug_set_flags(0)
