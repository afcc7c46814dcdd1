"""Oracle for core orthonormalisation and TT rounding.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  TT rounding "constitutes a fundamental
compression step applied subsequent to [rank-growing] operations ... to construct an
approximation subject to a specified error tolerance delta"; moving the block
index between cores is "one step of the TT rounding procedure".  Written out
after Oseledets (2011), "Tensor-Train Decomposition", Alg. 2 (TT-rounding): orthonormalise
right-to-left by QR, then truncate left-to-right by SVD with the per-core threshold
delta / sqrt(d - 1) * ||T||_F.  numpy's Householder QR and LAPACK SVD are the library steps.

Conventions: cores (r_k, n_k, r_{k+1}), C order.  QR results are sign-normalised so that the
triangular factor has a non-negative diagonal (the unique thin QR of a full-rank matrix).
"""
from __future__ import annotations

import numpy as np


def qr_pos(M: np.ndarray):
    """Thin QR with diag(R) >= 0."""
    Q, R = np.linalg.qr(M)
    s = np.sign(np.diag(R))
    s[s == 0] = 1.0
    return Q * s, s[:, None] * R


def core_qr_left(core: np.ndarray):
    """core (rl, n, rr) = Q (rl, n, s) . R (s, rr), s = min(rl n, rr), Q^T Q = I over (rl, n)."""
    rl, n, rr = core.shape
    Q, R = qr_pos(core.reshape(rl * n, rr))
    return Q.reshape(rl, n, Q.shape[1]), R


def core_lq_right(core: np.ndarray):
    """core (rl, n, rr) = L (rl, s) . Q (s, n, rr), s = min(rl, n rr), Q Q^T = I over (n, rr)
    (L lower trapezoidal)."""
    rl, n, rr = core.shape
    Qt, Rt = qr_pos(core.reshape(rl, n * rr).T)
    return Rt.T, Qt.T.reshape(Qt.shape[1], n, rr)


def orthonormalise_left(cores):
    """Left-orthonormalise cores 0..d-2 (R carried into the next core)."""
    cores = [np.array(c, dtype=np.float64) for c in cores]
    for k in range(len(cores) - 1):
        Q, R = core_qr_left(cores[k])
        cores[k] = Q
        cores[k + 1] = np.tensordot(R, cores[k + 1], axes=(1, 0))
    return cores


def orthonormalise_right(cores):
    """Right-orthonormalise cores d-1..1 (L carried into the previous core)."""
    cores = [np.array(c, dtype=np.float64) for c in cores]
    for k in range(len(cores) - 1, 0, -1):
        L, Q = core_lq_right(cores[k])
        cores[k] = Q
        cores[k - 1] = np.tensordot(cores[k - 1], L, axes=(2, 0))
    return cores


def tt_round(cores, delta: float, max_rank: int | None = None):
    """TT rounding (Oseledets Alg. 2): returns rounded cores with
    ||T - round(T)||_F <= delta ||T||_F."""
    d = len(cores)
    cores = orthonormalise_right(cores)
    nrm = float(np.linalg.norm(cores[0]))
    thr = delta / np.sqrt(max(d - 1, 1)) * nrm
    for k in range(d - 1):
        rl, n, rr = cores[k].shape
        U, S, Vt = np.linalg.svd(cores[k].reshape(rl * n, rr), full_matrices=False)
        # smallest rank whose discarded tail has Frobenius norm <= thr
        tail = np.sqrt(np.cumsum(S[::-1] ** 2))[::-1]      # tail[i] = ||S[i:]||
        rnew = len(S)
        for i in range(1, len(S) + 1):
            if i == len(S) or tail[i] <= thr:
                rnew = i
                break
        if max_rank is not None:
            rnew = min(rnew, max_rank)
        cores[k] = U[:, :rnew].reshape(rl, n, rnew)
        SV = S[:rnew, None] * Vt[:rnew]
        cores[k + 1] = np.tensordot(SV, cores[k + 1], axes=(1, 0))
    return cores


def _svd_rank(S: np.ndarray, delta: float, max_rank: int | None) -> int:
    """Smallest s with ||S[s:]||_2 <= delta ||S||_2 (then capped at max_rank)."""
    thr = delta * float(np.linalg.norm(S))
    tail = np.sqrt(np.cumsum(S[::-1] ** 2))[::-1]      # tail[i] = ||S[i:]||
    s = len(S)
    for i in range(1, len(S) + 1):
        if i == len(S) or tail[i] <= thr:
            s = i
            break
    if max_rank:
        s = min(s, max_rank)
    return s


def block_move_right(Wk_hat, Wk1, delta: float = 0.0, max_rank: int | None = None):
    """Move the block index l of the Block-TT core Wk_hat (r0, n0, l, r1) into the next core
    Wk1 (r1, n1, r2) by one SVD step of TT rounding (Def. Block TT PAPER.md:294-300):
    Wk_hat[(a,i), (l,b)] = U S V^T, truncated to s; returns Wk = U_s (r0, n0, s) and
    Wk1_hat[s, j, l, c] = sum_b (S V^T)_s[s, (l, b)] Wk1[b, j, c]."""
    r0, n0, l, r1 = Wk_hat.shape
    M = np.asarray(Wk_hat, dtype=np.float64).reshape(r0 * n0, l * r1)
    U, S, Vt = np.linalg.svd(M, full_matrices=False)
    s = _svd_rank(S, delta, max_rank)
    C = (S[:s, None] * Vt[:s]).reshape(s, l, r1)
    return U[:, :s].reshape(r0, n0, s), np.einsum("slb,bjc->sjlc", C, Wk1)


def block_move_left(Wkm1, Wk_hat, delta: float = 0.0, max_rank: int | None = None):
    """Mirror: move l of Wk_hat (r1, n1, l, r2) into the previous core Wkm1 (r0, n0, r1):
    Wk_hat[(a,l), (j,c)] = U S V^T truncated to s; returns Wkm1_hat (r0, n0, l, s) =
    Wkm1 x (U S)_s and Wk = V^T_s (s, n1, r2)."""
    r1, n1, l, r2 = Wk_hat.shape
    M = np.asarray(Wk_hat, dtype=np.float64).transpose(0, 2, 1, 3).reshape(r1 * l, n1 * r2)
    U, S, Vt = np.linalg.svd(M, full_matrices=False)
    s = _svd_rank(S, delta, max_rank)
    C = (U[:, :s] * S[:s]).reshape(r1, l, s)
    return np.einsum("ajb,bls->ajls", Wkm1, C), Vt[:s].reshape(s, n1, r2)
