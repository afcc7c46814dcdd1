import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2509_11890_b200 as tt
for rows, c, kappa in [(256, 256, 1e2), (256, 256, 1e6), (256, 256, 1e10), (256, 256, 1e14), (64, 64, 1e14), (256,256,1e0)]:
    rng = np.random.default_rng(rows * 7 + c)
    k = min(rows, c)
    s = np.logspace(0, -np.log10(kappa), k)
    U = np.linalg.qr(rng.standard_normal((rows, k)))[0]
    V = np.linalg.qr(rng.standard_normal((c, k)))[0]
    B = (U * s) @ V.T
    BJ, J, sig, sw = tt.tt_debug_svd(torch.from_numpy(B).cuda())
    BJ = BJ.cpu().numpy(); sig = sig.cpu().numpy()
    G = BJ.T @ BJ
    d = np.sqrt(np.outer(np.diag(G), np.diag(G)))
    off = np.abs(G - np.diag(np.diag(G))) / np.where(d > 0, d, 1)
    got = np.sort(sig)[::-1]
    rel = np.abs(got - s) / s
    print(rows, c, kappa, 'sweeps', int(sw.cpu()[0]), 'max off', off.max(), 'worst rel sigma', rel.max(), 'at', rel.argmax(), flush=True)
