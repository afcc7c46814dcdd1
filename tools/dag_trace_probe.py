"""Per-unit timeline of one W34 DAG launch (tt_debug_dag_trace): per task its window, the
average wait / mainloop / epilogue+publish per unit, and the gaps along the chains."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 3
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
inp = ttgen.make_inputs(idx)
x = [torch.from_numpy(c).cuda() for c in inp.x]
A = [torch.from_numpy(c).cuda() for c in inp.A]
tt.tt_debug_set_dag(mode)
for _ in range(3):
    tt.tt_sweep_w34(x, A)
torch.cuda.synchronize()
buf = torch.zeros(5 * 200000, dtype=torch.int64, device="cuda")
tt.tt_debug_dag_trace(buf)
tt.tt_sweep_w34(x, A)
torch.cuda.synchronize()
nt, nu, u0 = tt.tt_debug_dag_trace(None)
tr = buf[: 5 * nu].view(nu, 5).cpu().numpy().astype(np.int64)
t0 = tr[:, 0].min()
tr[:, :4] -= t0
print(f"config {idx} mode {mode}: {nt} tasks, {nu} units, span {tr[:, 3].max() / 1e3:.1f} us, "
      f"SMs used {len(set(tr[:, 4].tolist()))}")
print(" task units  first_grab first_ready last_done  | wait  main  epi (us, mean per unit)")
for i in range(nt):
    a, b = u0[i], u0[i + 1]
    s = tr[a:b]
    print(f" {i:3d} {b - a:5d}  {s[:, 0].min() / 1e3:9.1f} {s[:, 1].min() / 1e3:9.1f} {s[:, 3].max() / 1e3:9.1f}"
          f"  | {np.mean(s[:, 1] - s[:, 0]) / 1e3:5.2f} {np.mean(s[:, 2] - s[:, 1]) / 1e3:5.2f} "
          f"{np.mean(s[:, 3] - s[:, 2]) / 1e3:5.2f}")
tt.tt_debug_set_dag(0)
