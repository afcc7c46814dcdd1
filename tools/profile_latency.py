"""Profiling driver for the latency-path kernels: one K = 1 GMRES(10) cycle at the config-3
interior shape (fused cluster orthogonalisation, gmres_orth_cluster_kernel) and one config-3
interface sweep (fused small boundary runs, small_chain_kernel)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

tt.tt_set_graph_cache(False)
a, al, N = 64, 16, 4
rng = np.random.default_rng(1)
g = lambda x: torch.from_numpy(x).cuda()
phL = g(rng.standard_normal((a, al, a)) / a)
phR = g(rng.standard_normal((a, al, a)) / a)
A = g(rng.standard_normal((al, N, N, al)) / np.sqrt(al * N))
F = g(rng.standard_normal((a, N, 1, a)))
tt.tt_local_gmres(phL, A, phR, F, m=10, cycles=1, tol=0.0)
inp = ttgen.make_inputs(3)
x = [g(c) for c in inp.x]
As = [g(c) for c in inp.A]
tt.tt_sweep_interfaces(x, As)
torch.cuda.synchronize()
