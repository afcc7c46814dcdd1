"""Dense brute-force constructions straight from the paper's definitions (test side only).

Written independently of oracle/ and of the CUDA path: these materialise the full objects
that the TT hot path never forms, so they can pin the oracle.  Orderings are C order
(first core most significant), reading A4 of DESIGN.md.

* full TT vector:  T(a_1..a_d) = T_1(a_1) ... T_d(a_d)            PAPER.md:233-236 (Def. TT)
* full TT matrix:  A(i;j) = A_1(i_1,j_1) ... A_d(i_d,j_d)
* interface matrices T^{<k}, T^{>k}
* frame matrix T_{!=k} = T^{<k} (x) I_{n_k} (x) T^{>k}
* projected operator X_{!=k}^T A X_{!=k}
"""
from __future__ import annotations

import numpy as np


def full_vector(cores) -> np.ndarray:
    """vec(T) in C order, by the product of core slices (Def. TT)."""
    v = np.ones((1, 1))
    for c in cores:
        r0, n, r1 = c.shape
        # v[(I), r0] @ c[r0, (n r1)]  -> [(I n), r1]
        v = (v @ c.reshape(r0, n * r1)).reshape(-1, r1)
    assert v.shape[1] == 1
    return v[:, 0].copy()


def full_matrix(cores) -> np.ndarray:
    """Dense TT matrix (rows = output multi-index, cols = input multi-index), Def. TT Matrix."""
    W = np.ones((1, 1, 1))  # (I, J, r)
    for c in cores:
        r0, ni, nj, r1 = c.shape
        I, J, _ = W.shape
        W = np.einsum("IJr,rijs->IiJjs", W, c).reshape(I * ni, J * nj, r1)
    assert W.shape[2] == 1
    return W[:, :, 0].copy()


def left_interface(cores, k: int) -> np.ndarray:
    """T^{<k} (0-based: product of cores 0..k-1) as (prod n_j, r_k); T^{<1} = 1."""
    v = np.ones((1, 1))
    for c in cores[:k]:
        r0, n, r1 = c.shape
        v = (v @ c.reshape(r0, n * r1)).reshape(-1, r1)
    return v


def right_interface(cores, k: int) -> np.ndarray:
    """T^{>k} (0-based: product of cores k+1..d-1) as (prod n_j, r_{k+1}); T^{>d} = 1."""
    v = np.ones((1, 1))  # (r, J)
    for c in reversed(cores[k + 1:]):
        r0, n, r1 = c.shape
        v = (c.reshape(r0 * n, r1) @ v).reshape(r0, -1)
    return v.T.copy()


def frame(cores, k: int) -> np.ndarray:
    """T_{!=k} = T^{<k} (x) I_{n_k} (x) T^{>k}."""
    n = cores[k].shape[1]
    return np.kron(np.kron(left_interface(cores, k), np.eye(n)), right_interface(cores, k))


def projected_operator(x_cores, A_full, k: int) -> np.ndarray:
    """X_{!=k}^T A X_{!=k}."""
    F = frame(x_cores, k)
    return F.T @ A_full @ F


def left_matrix_interface(A_cores, k: int) -> np.ndarray:
    """Partial TT-matrix product of operator cores 0..k-1: (I, J, R_k)."""
    W = np.ones((1, 1, 1))
    for c in A_cores[:k]:
        r0, ni, nj, r1 = c.shape
        I, J, _ = W.shape
        W = np.einsum("IJr,rijs->IiJjs", W, c).reshape(I * ni, J * nj, r1)
    return W


def right_matrix_interface(A_cores, k: int) -> np.ndarray:
    """Partial TT-matrix product of operator cores k..d-1: (R_k, I, J)."""
    W = np.ones((1, 1, 1))  # (r, I, J)
    for c in reversed(A_cores[k:]):
        r0, ni, nj, r1 = c.shape
        _, I, J = W.shape
        W = np.einsum("rijs,sIJ->riIjJ", c, W).reshape(r0, ni * I, nj * J)
    return W


def phiL_dense(x_cores, A_cores, k: int) -> np.ndarray:
    """Phi^L after cores 0..k-1: [b', beta, b] = sum X^{<}[I,b'] A^{<}[I,J,beta] X^{<}[J,b]."""
    X = left_interface(x_cores, k)
    A = left_matrix_interface(A_cores, k)
    return np.einsum("Ip,IJs,Jq->psq", X, A, X)


def phiR_dense(x_cores, A_cores, k: int) -> np.ndarray:
    """Phi^R of cores k..d-1: [a', alpha, a] = sum X^{>=}[a',I] A^{>=}[alpha,I,J] X^{>=}[a,J]."""
    # right interface of cores k..d-1 as (r_k, prod n)
    v = np.ones((1, 1))
    for c in reversed(x_cores[k:]):
        r0, n, r1 = c.shape
        v = (c.reshape(r0 * n, r1) @ v).reshape(r0, -1)
    A = right_matrix_interface(A_cores, k)
    return np.einsum("pI,sIJ,qJ->psq", v, A, v)


def unvec_tt_dense(v_full: np.ndarray, d: int, n: int) -> np.ndarray:
    """vec_TT index (a_1,b_1,...,a_d,b_d) -> matrix M[(a_1..a_d),(b_1..b_d)]."""
    t = v_full.reshape([n] * (2 * d))
    perm = list(range(0, 2 * d, 2)) + list(range(1, 2 * d, 2))
    return t.transpose(perm).reshape(n ** d, n ** d)


def vec_tt_dense(M: np.ndarray, d: int, n: int) -> np.ndarray:
    """Inverse of unvec_tt_dense."""
    t = M.reshape([n] * (2 * d))
    perm = []
    for k in range(d):
        perm += [k, d + k]
    return t.transpose(perm).reshape(-1)


def rel_fro(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)
