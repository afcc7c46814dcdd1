"""Device time (CUDA-graph replay, median) of the bench's NEXT-row workloads at the config-5
interior core: KKT block action (9 K = 1 matvecs), LOBPCG nb = 8 x 20 iterations (standard and
generalised) -- the same inputs and timing as bench.py, without the rest of the bench.
python tools/next_rows_time.py [kkt|lobpcg|all] [debug_flags]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
from bench import time_sweep  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dev = torch.device("cuda")
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)   # graph.replay() runs on the current stream (as in bench.py)
rl = rr = 256
nn, Rl, Rr = 4, 36, 36
f_local = 2.0 * (rl * Rl * rl * nn * rr + Rl * nn * nn * Rr * rl * rr + rl * nn * Rr * rr * rr)
p64 = 37.18
tt.tt_debug_set_flags(flags)
if what in ("kkt", "all"):
    gen = torch.Generator(device=dev).manual_seed(11)
    rnd = lambda *sh: torch.randn(*sh, dtype=torch.float64, device=dev, generator=gen)
    ops = [(rnd(rl, Rl, rl), rnd(Rl, nn, nn, Rr), rnd(rr, Rr, rr)) for _ in range(8)]
    terms = [(0, 0, 0, -1, -1.0), (0, 1, 1, -1, 1.0), (1, 0, 2, -1, -1.0),
             (1, 2, 3, -1, 1.0), (2, 0, 4, -1, 1.0), (2, 1, 5, 6, 1.0), (2, 2, 5, 7, 1.0)]
    Xk = rnd(rl, nn, 3, rr)
    Yk = torch.empty_like(Xk)
    wsk = torch.empty(tt.tt_block_local_matvec_workspace_size(rl, nn, rr, [Rl] * 8, [Rr] * 8),
                      dtype=torch.uint8, device=dev)
    t = time_sweep(tt, lambda st: tt.tt_block_local_matvec(ops, terms, Xk, Yk, workspace=wsk,
                                                          stream=st), stream, dev, reps=5)
    f9 = 9 * f_local
    print(f"kkt: graph {t['graph_ms_median']:.3f} ms eager {t['eager_ms_median']:.3f} ms "
          f"{f9 / t['graph_ms_median'] / 1e9:.2f} TFLOP/s = {f9 / t['graph_ms_median'] / 1e9 / p64:.3f} of P64",
          flush=True)
if what in ("lobpcg", "all"):
    gen = torch.Generator(device=dev).manual_seed(12)
    rnd = lambda *sh: torch.randn(*sh, dtype=torch.float64, device=dev, generator=gen)
    sym_if = lambda r, R: (lambda t: (t + t.transpose(0, 2)) / 2)(rnd(r, R, r))
    sym_core = lambda: (lambda t: (t + t.transpose(1, 2)) / 2)(rnd(Rl, nn, nn, Rr))
    opA = (sym_if(rl, Rl), sym_core(), sym_if(rr, Rr))
    pLB, ALB, pRB = 0.1 * sym_if(rl, Rl), 0.1 * sym_core(), 0.1 * sym_if(rr, Rr)
    pLB[:, 0, :] += torch.eye(rl, dtype=torch.float64, device=dev)
    pRB[:, 0, :] += torch.eye(rr, dtype=torch.float64, device=dev)
    ALB[0, :, :, 0] = torch.eye(nn, dtype=torch.float64, device=dev)
    ALB[0, :, :, 1:] = 0.0
    ALB[1:, :, :, 0] = 0.0
    opB = (pLB, ALB, pRB)
    nb_l, its_l = 8, 20
    for name, oB in (("standard", None), ("generalised", opB)):
        X0 = rnd(rl, nn, nb_l, rr)
        Xl = X0.clone()
        RlB, RrB = (Rl, Rr) if oB is not None else (0, 0)
        wsl = torch.empty(tt.tt_local_lobpcg_workspace_size(rl, nn, rr, Rl, Rr, RlB, RrB, nb_l),
                          dtype=torch.uint8, device=dev)
        bufs = [torch.empty(nb_l, dtype=torch.float64, device=dev) for _ in range(2)]
        itl = torch.empty(1, dtype=torch.int64, device=dev)
        stl = torch.empty(1, dtype=torch.float64, device=dev)

        def lob_run(st, oB=oB, Xl=Xl, X0=X0, wsl=wsl, bufs=bufs, itl=itl, stl=stl):
            Xl.copy_(X0)
            tt.tt_local_lobpcg(opA, Xl, opB=oB, maxiter=its_l, tol=0.0, lam=bufs[0], res=bufs[1],
                               iters=itl, step=stl, workspace=wsl, stream=st, refresh=20)
        t = time_sweep(tt, lob_run, stream, dev, reps=3)
        nops = 2 if oB is not None else 1
        nblocks = 1 + its_l + 2 * ((its_l - 1) // 20)
        mv_f = nops * nblocks * nb_l * f_local
        print(f"lobpcg {name}: {t['graph_ms_median'] / its_l:.3f} ms/iteration, "
              f"{mv_f / t['graph_ms_median'] / 1e9 / p64:.3f} of P64 (matvec flops / total time), "
              f"lam0 {bufs[0][0].item():.10f}", flush=True)
tt.tt_debug_set_flags(0)
