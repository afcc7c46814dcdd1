"""One eager left-interface chain at config 4 (after warm-up), for an ncu launch list."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
inp = ttgen.make_inputs(idx)
x = [torch.from_numpy(c).cuda() for c in inp.x]
A = [torch.from_numpy(c).cuda() for c in inp.A]
tt.tt_set_graph_cache(False)
pl, pr = tt.alloc_interfaces(x, A), tt.alloc_interfaces(x, A)
for _ in range(2):
    tt.tt_sweep_interfaces(x, A, pl, pr, tt.TT_SWEEP_LEFT)
torch.cuda.synchronize()
