"""Oracle for the matrix-free local solve: restarted GMRES(m) and its
"accelerated" variant LGMRES(m, k).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The paper solves the projected local
systems "in a matrix-free fashion via GMRES, i.e. we do not explicitly form the projected
operators ... but instead perform the constituent multiplications sequentially ... we employ
the accelerated GMRES method [Baker2005]" (§3.3); the operator action is the
oracle's local matvec (tt_oracle_local_matvec).

GMRES is written out step by step in the textbook form (Saad, Iterative Methods for Sparse
Linear Systems, Alg. 6.9: Arnoldi with modified Gram-Schmidt, Givens rotations on the
Hessenberg matrix, back substitution), plain numpy, one right-hand side at a time.  The
acceleration follows Baker, Jessup & Manteuffel (2005), "A technique for accelerating the
convergence of restarted GMRES": each restart cycle's search space is augmented with the
k most recent error approximations z_j = x_j - x_{j-1} (the previous cycles' corrections),
i.e. the flexible Arnoldi relation A [v_1..v_m, z_1..z_k] = V_{m+k+1} Hbar is built by
orthonormalising A v_i (i <= m) and then A z_j against the growing orthonormal basis, the
residual is minimised over x + span[v_1..v_m, z_1..z_k], and the new correction becomes the
newest z.  k = 0 is plain GMRES(m).
"""
from __future__ import annotations

import numpy as np

from . import local_matvec


def gmres(apply, f: np.ndarray, x0: np.ndarray, m: int, cycles: int, tol: float, k: int = 0):
    """Restarted GMRES(m) (k = 0) or LGMRES(m, k) for apply(x) = f on flat float64 vectors.

    Returns (x, rel_res, iters): the iterate after `cycles` restart cycles (or earlier
    convergence), the final Givens residual estimate |g_{s+1}| / ||f|| (the true relative
    residual at the start of the cycle if the cycle did not run), and the total number of
    Arnoldi steps.  Convergence test: |g_{i+1}| <= tol * ||f||.
    """
    f = np.asarray(f, dtype=np.float64).ravel()
    x = np.asarray(x0, dtype=np.float64).ravel().copy()
    fnorm = float(np.linalg.norm(f))
    if fnorm == 0.0:
        return np.zeros_like(x), 0.0, 0
    iters = 0
    rel = None
    Z = []                                              # newest first, unit norm
    for _ in range(cycles):
        r = f - apply(x)
        beta = float(np.linalg.norm(r))
        rel = beta / fnorm
        if rel <= tol:
            break
        s = m + len(Z)                                  # search-space dimension
        V = np.zeros((s + 1, x.size))
        Wcols = []                                      # the vectors multiplied by A
        H = np.zeros((s + 1, s))
        cs = np.zeros(s)
        sn = np.zeros(s)
        g = np.zeros(s + 1)
        g[0] = beta
        V[0] = r / beta
        kk = 0
        for i in range(s):
            wi = V[i] if i < m else Z[i - m]
            Wcols.append(wi)
            w = apply(wi)
            for l in range(i + 1):                      # modified Gram-Schmidt
                H[l, i] = float(np.dot(w, V[l]))
                w = w - H[l, i] * V[l]
            H[i + 1, i] = float(np.linalg.norm(w))
            if H[i + 1, i] != 0.0:
                V[i + 1] = w / H[i + 1, i]
            for l in range(i):                          # previous rotations on column i
                t = cs[l] * H[l, i] + sn[l] * H[l + 1, i]
                H[l + 1, i] = -sn[l] * H[l, i] + cs[l] * H[l + 1, i]
                H[l, i] = t
            den = float(np.hypot(H[i, i], H[i + 1, i]))  # new rotation zeroes H[i+1, i]
            cs[i] = H[i, i] / den
            sn[i] = H[i + 1, i] / den
            H[i, i] = den
            H[i + 1, i] = 0.0
            g[i + 1] = -sn[i] * g[i]
            g[i] = cs[i] * g[i]
            kk = i + 1
            iters += 1
            rel = abs(g[i + 1]) / fnorm
            if rel <= tol:
                break
        y = np.zeros(kk)                                # back substitution H[:kk,:kk] y = g[:kk]
        for l in range(kk - 1, -1, -1):
            y[l] = (g[l] - float(np.dot(H[l, l + 1:kk], y[l + 1:kk]))) / H[l, l]
        corr = np.zeros_like(x)
        for l in range(kk):
            corr = corr + y[l] * Wcols[l]
        x = x + corr
        if k > 0:                                       # newest error approximation first
            cn = float(np.linalg.norm(corr))
            if cn > 0.0:
                Z = [corr / cn] + Z[:k - 1]
        if rel <= tol:
            break
    return x, rel, iters


def local_gmres_batched(phiL, A, phiR, F, X0, m: int, cycles: int, tol: float, k: int = 0):
    """(L)GMRES on the projected local operator (tt_oracle_local_matvec) for every column of
    a Block-TT right-hand side F (rl, n, K, rr); columns are independent systems."""
    F = np.ascontiguousarray(F, dtype=np.float64)
    X0 = np.ascontiguousarray(X0, dtype=np.float64)
    rl, n, K, rr = F.shape
    shape = (rl, n, rr)
    apply = lambda v: local_matvec(phiL, A, phiR, v.reshape(shape)).ravel()
    X = np.empty_like(F)
    rel = np.empty(K)
    its = np.empty(K, dtype=np.int64)
    for j in range(K):
        x, rel[j], its[j] = gmres(apply, F[:, :, j, :].ravel(), X0[:, :, j, :].ravel(), m,
                                  cycles, tol, k)
        X[:, :, j, :] = x.reshape(shape)
    return X, rel, its
