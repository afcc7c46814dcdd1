"""W34 (configs 3 / 4) split into its parts, each replayed from a CUDA graph: the two
interface chains (tt_sweep_interfaces, left and right concurrently), the d matvecs, and the
whole workload.  usage: python tools/w34_parts.py [config ...]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402


def graph_ms(fn, reps=20):
    s = torch.cuda.Stream()
    fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            fn(s)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for idx in [int(a) for a in (sys.argv[1:] or ["3", "4"])]:
    inp = ttgen.make_inputs(idx)
    x = [torch.from_numpy(c).cuda() for c in inp.x]
    A = [torch.from_numpy(c).cuda() for c in inp.A]
    pl, pr = tt.alloc_interfaces(x, A), tt.alloc_interfaces(x, A)
    y = [torch.empty_like(c) for c in x]
    tr = tt._Train(x, A)
    ws = torch.empty(tt.tt_sweep_workspace_size(tr), dtype=torch.uint8, device="cuda")
    wsm = torch.empty(max(tt.tt_local_matvec_workspace_size(c.shape[0], c.shape[1], c.shape[2],
                                                            a.shape[0], a.shape[3], 1)
                          for c, a in zip(x, A)), dtype=torch.uint8, device="cuda")

    def chains(s):
        tt.tt_sweep_interfaces(x, A, pl, pr, workspace=ws, stream=s)

    def left(s):
        tt.tt_sweep_interfaces(x, A, pl, None, directions=tt.TT_SWEEP_LEFT, workspace=ws, stream=s)

    def mvs(s):
        for k in range(len(x)):
            tt.tt_local_matvec(pl[k], A[k], pr[k + 1], x[k], y[k], workspace=wsm, stream=s)

    def w34(s):
        chains(s)
        mvs(s)
    ws34 = torch.empty(tt.tt_sweep_w34_workspace_size(tr), dtype=torch.uint8, device="cuda")

    def w34_dag(s):
        tt.tt_sweep_w34(x, A, pl, pr, y, workspace=ws34, stream=s)
    res = {name: graph_ms(f) for name, f in (("both_chains", chains), ("left_chain", left),
                                             ("matvecs", mvs), ("w34", w34),
                                             ("w34_dag", w34_dag))}
    tt.tt_debug_set_flags(2048)   # chains at the lowest priority (A/B)
    res["w34_dag_lowprio_side"] = graph_ms(w34_dag)
    tt.tt_debug_set_flags(4096)   # plain launches instead of PDL (A/B)
    res["w34_dag_no_pdl"] = graph_ms(w34_dag)
    res["left_chain_no_pdl"] = graph_ms(left)
    tt.tt_debug_set_flags(8192)   # default tile policy for small GEMMs (A/B)
    res["w34_dag_no_latency_tiles"] = graph_ms(w34_dag)
    res["left_chain_no_latency_tiles"] = graph_ms(left)
    tt.tt_debug_set_flags(0)
    print(f"config {idx}: " + "  ".join(f"{k} {v:.3f} ms" for k, v in res.items()), flush=True)
