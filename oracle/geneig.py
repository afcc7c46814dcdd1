"""Oracle for the step-length local eigenproblem.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The paper computes the optimal step length
from local generalised eigenproblems:

    max_{E_k} vec(E_k)^T E_{!=k}^T dM E_{!=k} vec(E_k)   s.t.   vec(E_k)^T E_{!=k}^T M E_{!=k} vec(E_k) = 1,

"A sparse eigenvalue solver with a Cholesky-based reduction finds the largest eigenvalue", and
notes the matrix-free alternative LOBPCG.  An iterative eigensolver converges to
a result with a plain definition -- the largest eigenpairs of the projected pencil -- so the
oracle is that definition written out:

1. the projected operator as a dense matrix, entry by entry from master formula (M)
   (X_{!=k}^T A X_{!=k}), rows (a', i, b'), columns (a, j, b);
2. the Cholesky-based reduction named by the paper: L_B = C C^T, S = C^{-1} L_A C^{-T}
   (numpy Cholesky and two triangular solves), eigenpairs of the symmetric S (LAPACK eigh, a
   library primitive), back-transformation v = C^{-T} u (L_B-orthonormal eigenvectors);
3. the step length (reading R12 of DESIGN.md): alpha = min(1, 1 / lam_max) when lam_max > 0,
   else 1, where lam_max is the largest eigenvalue of the pencil (-dM, M).  X + alpha dX stays
   positive semidefinite exactly for alpha <= 1 / lam_max (PAPER.md:561-563 garbles the ratio;
   the cap at 1 is PAPER.md:564).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg


def local_operator_dense(phiL: np.ndarray, A: np.ndarray, phiR: np.ndarray) -> np.ndarray:
    """L[(a',i,b'), (a,j,b)] = sum_{alpha,beta} phiL[a',alpha,a] A[alpha,i,j,beta] phiR[b',beta,b]."""
    rl, n, rr = phiL.shape[0], A.shape[1], phiR.shape[0]
    L = np.einsum("pxa,xijy,qyb->piqajb", phiL, A, phiR)
    return L.reshape(rl * n * rr, rl * n * rr)


def block_columns(X: np.ndarray) -> np.ndarray:
    """Block-TT core (rl, n, nb, rr) -> matrix of its nb vectorised columns (rl n rr, nb)."""
    rl, n, nb, rr = X.shape
    return np.ascontiguousarray(X.transpose(0, 1, 3, 2)).reshape(rl * n * rr, nb)


def columns_block(V: np.ndarray, rl: int, n: int, rr: int) -> np.ndarray:
    nb = V.shape[1]
    return np.ascontiguousarray(V.reshape(rl, n, rr, nb).transpose(0, 1, 3, 2))


def geneig_dense(LA: np.ndarray, LB: np.ndarray | None, nb: int):
    """nb largest eigenpairs of the symmetric pencil (LA, LB), LB SPD (None = identity), by the
    Cholesky-based reduction.  Returns (lam descending (nb,), V (n, nb) with V^T LB V = I)."""
    LA = 0.5 * (LA + LA.T)
    if LB is None:
        w, U = np.linalg.eigh(LA)
        idx = np.argsort(-w, kind="stable")[:nb]
        return w[idx], U[:, idx]
    LB = 0.5 * (LB + LB.T)
    C = np.linalg.cholesky(LB)                                    # LB = C C^T
    Y = scipy.linalg.solve_triangular(C, LA, lower=True)          # C^{-1} LA
    S = scipy.linalg.solve_triangular(C, Y.T, lower=True).T       # C^{-1} LA C^{-T}
    S = 0.5 * (S + S.T)
    w, U = np.linalg.eigh(S)
    idx = np.argsort(-w, kind="stable")[:nb]
    V = scipy.linalg.solve_triangular(C.T, U[:, idx], lower=False)  # v = C^{-T} u
    return w[idx], V


def local_geneig(opA, opB, nb: int):
    """nb largest eigenpairs of the projected pencil; opA, opB = (phiL, A, phiR) (opB None: I)."""
    LA = local_operator_dense(*opA)
    LB = None if opB is None else local_operator_dense(*opB)
    return geneig_dense(LA, LB, nb)


def step_length(lam_max: float) -> float:
    """alpha = min(1, 1/lam_max) for lam_max > 0 (the pencil (-dM, M)), else 1."""
    return min(1.0, 1.0 / lam_max) if lam_max > 0.0 else 1.0
