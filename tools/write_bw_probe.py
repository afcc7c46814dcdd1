"""HBM write-only bandwidth (the roof of the write-bound apply H8) vs copy bandwidth, and the
config-5 apply alone: torch fill_ (store-only kernel), cudaMemsetAsync, tensor copy."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_11890_b200 as tt  # noqa: E402
import ttgen  # noqa: E402


def t(fn, reps=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


n = 1 << 30   # 8 GiB of doubles
a = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty(n // 2, dtype=torch.float64, device="cuda")
c = torch.empty(n // 2, dtype=torch.float64, device="cuda")
ms = t(lambda: a.fill_(1.0))
print(f"fill_ (write only): {8 * n / ms / 1e6:.0f} GB/s")
ms = t(lambda: a.zero_())
print(f"zero_ (memset):     {8 * n / ms / 1e6:.0f} GB/s")
ms = t(lambda: b.copy_(c))
print(f"copy (read+write):  {2 * 8 * (n // 2) / ms / 1e6:.0f} GB/s")
del a, b, c
torch.cuda.empty_cache()
inp = ttgen.make_inputs(5)
x = [torch.from_numpy(v).cuda() for v in inp.x]
A = [torch.from_numpy(v).cuda() for v in inp.A]
z = tt.tt_operator_apply(x, A)
p = tt.prepare(tt.tt_operator_apply, x, A, z)
ms = t(lambda: p())
nb = sum(v.numel() * 8 for v in z) + sum(v.numel() * 8 for v in x) + sum(v.numel() * 8 for v in A)
print(f"apply config 5: {ms:.3f} ms, {nb / ms / 1e6:.0f} GB/s")
for flags, name in [(0, "default: row-block kernel"), (1 << 27, "register-blocked kernel (debug bit 27)")]:
    tt.tt_debug_set_flags(flags)
    p = tt.prepare(tt.tt_operator_apply, x, A, z)
    ms = t(lambda: p())
    print(f"apply config 5 [{name}]: {ms:.3f} ms, {nb / ms / 1e6:.0f} GB/s", flush=True)
tt.tt_debug_set_flags(0)
