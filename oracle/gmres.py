"""Oracle for the matrix-free local solve: restarted GMRES(m).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The paper solves the projected local
systems "in a matrix-free fashion via GMRES, i.e. we do not explicitly form the projected
operators ... but instead perform the constituent multiplications sequentially"
(§3.3); the operator action is the oracle's local matvec
(tt_oracle_local_matvec).  GMRES itself is written out step by step in the
textbook form (Saad, Iterative Methods for Sparse Linear Systems, Alg. 6.9: Arnoldi with
modified Gram-Schmidt, Givens rotations on the Hessenberg matrix, back substitution),
plain numpy, one right-hand side at a time.

The paper's "accelerated" variant (Baker et al. 2005, LGMRES) is not reproduced here; the
GPU side implements the same plain GMRES(m).
"""
from __future__ import annotations

import numpy as np

from . import local_matvec


def gmres(apply, f: np.ndarray, x0: np.ndarray, m: int, cycles: int, tol: float):
    """Restarted GMRES(m) for apply(x) = f on flat float64 vectors.

    Returns (x, rel_res, iters): the iterate after `cycles` restart cycles (or earlier
    convergence), the final Givens residual estimate |g_{k+1}| / ||f||, and the total number
    of Arnoldi steps taken.  Convergence test: |g_{i+1}| <= tol * ||f||.
    """
    f = np.asarray(f, dtype=np.float64).ravel()
    x = np.asarray(x0, dtype=np.float64).ravel().copy()
    fnorm = float(np.linalg.norm(f))
    if fnorm == 0.0:
        return np.zeros_like(x), 0.0, 0
    iters = 0
    rel = None
    for _ in range(cycles):
        r = f - apply(x)
        beta = float(np.linalg.norm(r))
        rel = beta / fnorm
        if rel <= tol:
            break
        V = np.zeros((m + 1, x.size))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        k = 0
        for i in range(m):
            w = apply(V[i])
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
            k = i + 1
            iters += 1
            rel = abs(g[i + 1]) / fnorm
            if rel <= tol:
                break
        y = np.zeros(k)                                 # back substitution H[:k,:k] y = g[:k]
        for l in range(k - 1, -1, -1):
            y[l] = (g[l] - float(np.dot(H[l, l + 1:k], y[l + 1:k]))) / H[l, l]
        x = x + V[:k].T @ y
        if rel <= tol:
            break
    return x, rel, iters


def local_gmres_batched(phiL, A, phiR, F, X0, m: int, cycles: int, tol: float):
    """GMRES(m) on the projected local operator (tt_oracle_local_matvec) for every column
    of a Block-TT right-hand side F (rl, n, K, rr); columns are independent systems."""
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
                                  cycles, tol)
        X[:, :, j, :] = x.reshape(shape)
    return X, rel, its
