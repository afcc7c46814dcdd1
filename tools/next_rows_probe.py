"""One run of a NEXT-row workload at the config-5 interior-core size, for ncu launch lists
(python tools/next_rows_probe.py gmres|lobpcg|kkt|round|w34 [config])."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

what = sys.argv[1]
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(5)
rnd = lambda *sh: torch.randn(*sh, dtype=torch.float64, device=dev, generator=g)
a = b = 256
n, al, be, K = 4, 36, 36, 32
if what == "gmres":
    phiL, A, phiR, F = rnd(a, al, a), rnd(al, n, n, be), rnd(b, be, b), rnd(a, n, K, b)
    tt.tt_local_gmres(phiL, A, phiR, F, m=10, cycles=1, tol=0.0)
elif what == "lobpcg":
    sym = lambda t: (t + t.transpose(0, 2)) / 2
    opA = (sym(rnd(a, al, a)), (lambda t: (t + t.transpose(1, 2)) / 2)(rnd(al, n, n, be)),
           sym(rnd(b, be, b)))
    tt.tt_local_lobpcg(opA, rnd(a, n, 8, b), maxiter=5, tol=0.0)
elif what == "kkt":
    ops = [(rnd(a, al, a), rnd(al, n, n, be), rnd(b, be, b)) for _ in range(8)]
    terms = [(0, 0, 0, -1, -1.0), (0, 1, 1, -1, 1.0), (1, 0, 2, -1, -1.0),
             (1, 2, 3, -1, 1.0), (2, 0, 4, -1, 1.0), (2, 1, 5, 6, 1.0), (2, 2, 5, 7, 1.0)]
    tt.tt_block_local_matvec(ops, terms, rnd(a, n, 3, b))
elif what == "round":
    inp = ttgen.make_inputs(5, with_block=False)
    tt.tt_round([torch.from_numpy(c).to(dev) for c in inp.x], 1e-4)
elif what == "w34":
    inp = ttgen.make_inputs(int(sys.argv[2]) if len(sys.argv) > 2 else 4)
    tt.tt_sweep_w34([torch.from_numpy(c).to(dev) for c in inp.x],
                    [torch.from_numpy(c).to(dev) for c in inp.A])
torch.cuda.synchronize()
print(what, "launches", tt.tt_last_launch_count())
