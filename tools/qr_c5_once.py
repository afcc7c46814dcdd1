"""One right orthonormalisation of the config-5 train (1024 x 256 QRs), for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

x = [torch.from_numpy(c).cuda() for c in ttgen.make_inputs(5).x]
tt.tt_orthonormalise(x, tt.TT_SWEEP_RIGHT)
torch.cuda.synchronize()
