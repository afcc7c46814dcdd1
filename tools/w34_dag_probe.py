"""W34 (tt_sweep_w34) per config: DAG executor vs stream version, eager and CUDA-graph replay."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402


def timeit(fn, reps=30):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2], ts[0]


for idx in [int(a) for a in (sys.argv[1:] or ["1", "2", "3", "4"])]:
    inp = ttgen.make_inputs(idx)
    x = [torch.from_numpy(c).cuda() for c in inp.x]
    A = [torch.from_numpy(c).cuda() for c in inp.A]
    tr = tt._Train(x, A)
    ws = torch.empty(tt.tt_sweep_w34_workspace_size(tr), dtype=torch.uint8, device="cuda")
    pl, pr = tt.alloc_interfaces(x, A), tt.alloc_interfaces(x, A)
    y = [torch.zeros_like(c) for c in x]
    ref = None
    for mode in (0, 1, 2, 9):
        tt.tt_set_graph_cache(mode != 9)
        tt.tt_debug_set_dag(0 if mode == 9 else mode)
        s = torch.cuda.Stream()
        call = lambda: tt.tt_sweep_w34(x, A, pl, pr, y, workspace=ws, stream=s)
        if mode == 0:   # prepared call: one ctypes call per sweep
            call = tt.prepare(tt.tt_sweep_w34, x, A, pl, pr, y, workspace=ws, stream=s)
        with torch.cuda.stream(s):
            for _ in range(3):
                call()
        torch.cuda.synchronize()
        out = [c.clone() for c in y + pl + pr]
        if ref is None:
            ref = out
        err = max(float((a - b).norm() / max(b.norm(), 1e-300)) for a, b in zip(out, ref))
        with torch.cuda.stream(s):
            eager = timeit(call)
            import time
            torch.cuda.synchronize()
            h0 = time.perf_counter()
            for _ in range(20):
                call()
            host_us = (time.perf_counter() - h0) / 20 * 1e6
            torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                call()
        graph = timeit(g.replay)
        print(f"config {idx} dag={mode:2d}: eager {eager[0]*1e3:8.1f} us (best {eager[1]*1e3:8.1f})  "
              f"graph {graph[0]*1e3:8.1f} us (best {graph[1]*1e3:8.1f})  host {host_us:7.1f} us/call  "
              f"rel-diff vs stream {err:.1e}",
              flush=True)
    tt.tt_debug_set_dag(0)
