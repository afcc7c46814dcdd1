"""LOBPCG at the bench's interior-core size (config 5: a = b = 256, N = 4, R = 36, nb = 8):
a few iterations, for an ncu launch list (python tools/lobpcg_probe.py [iters] [generalised])."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402

its = int(sys.argv[1]) if len(sys.argv) > 1 else 5
gen_b = len(sys.argv) > 2 and sys.argv[2] == "1"
dev = torch.device("cuda")
rl = rr = 256
nn, Rl, Rr, nb = 4, 36, 36, 8
g = torch.Generator(device=dev).manual_seed(12)
rnd = lambda *sh: torch.randn(*sh, dtype=torch.float64, device=dev, generator=g)
sym_if = lambda r, R: (lambda t: (t + t.transpose(0, 2)) / 2)(rnd(r, R, r))
sym_core = lambda: (lambda t: (t + t.transpose(1, 2)) / 2)(rnd(Rl, nn, nn, Rr))
opA = (sym_if(rl, Rl), sym_core(), sym_if(rr, Rr))
opB = None
if gen_b:
    pLB, ALB, pRB = 0.1 * sym_if(rl, Rl), 0.1 * sym_core(), 0.1 * sym_if(rr, Rr)
    pLB[:, 0, :] += torch.eye(rl, dtype=torch.float64, device=dev)
    pRB[:, 0, :] += torch.eye(rr, dtype=torch.float64, device=dev)
    ALB[0, :, :, 0] = torch.eye(nn, dtype=torch.float64, device=dev)
    ALB[0, :, :, 1:] = 0.0
    ALB[1:, :, :, 0] = 0.0
    opB = (pLB, ALB, pRB)
X = rnd(rl, nn, nb, rr)
X, lam, res, it, step = tt.tt_local_lobpcg(opA, X, opB=opB, maxiter=its, tol=0.0)
torch.cuda.synchronize()
print("lam", lam.cpu().numpy(), "res", res.cpu().numpy().max(), "launches", tt.tt_last_launch_count())
