"""Sweep counts of the cluster Jacobi SVD (tt_debug_svd) on R^T of B = U diag(s) V^T, s graded
to 1/kappa, against a numpy model of the same parallel ordering (tools/README.md)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2509_11890_b200 as tt

def run(n, kappa, pre=True, seed=0):
    rng = np.random.default_rng(seed)
    s = np.logspace(0, -np.log10(kappa), n)
    U = np.linalg.qr(rng.standard_normal((n, n)))[0]
    V = np.linalg.qr(rng.standard_normal((n, n)))[0]
    B = (U * s) @ V.T
    if pre:
        B = np.ascontiguousarray(np.linalg.qr(B)[1].T)
    BJ, J, sig, sw = tt.tt_debug_svd(torch.from_numpy(B).cuda())
    torch.cuda.synchronize()
    sig = np.sort(sig.cpu().numpy())[::-1]
    rel = np.abs(sig - s) / s
    return int(sw.cpu()[0]), rel[s > 1e-13].max()

for n in (() if len(sys.argv) > 1 else (64, 128, 256)):
    for kappa in (1e8, 1e10, 1e12, 1e13, 1e14, 1e15):
        print(n, kappa, *run(n, kappa), flush=True)
if len(sys.argv) > 1:
    for seed in [2048, 1, 2, 3, 4, 5, 6, 7]:
        print('seed', seed, *run(256, 1e14, seed=seed), *run(256, 1e15, seed=seed), flush=True)
