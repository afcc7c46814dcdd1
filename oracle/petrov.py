"""Oracle for the Petrov-Galerkin local operations and the AMEn enrichment (SURVEY.md §8(f)
row 3).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  With two trains -- a bra train Z and a
ket train X on the same modes -- the projected operator Z_{!=k}^T A X_{!=k} (PAPER.md:289-292
with the bra frame replaced), the projected right-hand side X_{!=k}^T vec(B) of the local
system (an identity operator and the right-hand side train B as ket) and the
residual core of AMEn ("enrichment of the TT cores by TT cores of the approximate residual,
as in the AMEn algorithm"; Dolgov & Savostyanov 2014) are the master formulas
(M), (IL), (IR) of SURVEY.md §8 with the bra ranks decoupled from the ket ranks.  Written as
the plain sums, evaluated as the three products of PAPER.md:526 (numpy tensordot is the
library contraction); interfaces are [bra, op, ket].
"""
from __future__ import annotations

import numpy as np

from .rounding import block_move_right


def local_matvec_pg(phiL, A, phiR, X):
    """Y[a',i,(m,)b'] = sum phiL[a',al,a] A[al,i,j,be] phiR[b',be,b] X[a,j,(m,)b], evaluated as
    the three products of PAPER.md:526 (each a two-operand contraction)."""
    Xb = X[:, :, None, :] if X.ndim == 3 else X
    T1 = np.tensordot(phiL, Xb, axes=(2, 0))                    # a' al | j m b
    T2 = np.tensordot(T1, A, axes=([1, 2], [0, 2]))             # a' m b | i be
    Y = np.tensordot(T2, phiR, axes=([2, 4], [2, 1]))           # a' m i | b'
    Y = Y.transpose(0, 2, 1, 3)                                 # a' i m b'
    return np.ascontiguousarray(Y[:, :, 0, :] if X.ndim == 3 else Y)


def interface_left_pg(phiL, A, x_bra, x_ket):
    """phiL_next[b',be,b] = sum x_bra[a',i,b'] phiL[a',al,a] A[al,i,j,be] x_ket[a,j,b]."""
    T1 = np.tensordot(phiL, x_ket, axes=(2, 0))                 # a' al | j b
    T2 = np.tensordot(T1, A, axes=([1, 2], [0, 2]))             # a' b | i be
    return np.ascontiguousarray(np.tensordot(x_bra, T2, axes=([0, 1], [0, 2])).transpose(0, 2, 1))


def interface_right_pg(phiR, A, x_bra, x_ket):
    """phiR_prev[a',al,a] = sum x_bra[a',i,b'] A[al,i,j,be] phiR[b',be,b] x_ket[a,j,b]."""
    T1 = np.tensordot(x_ket, phiR, axes=(2, 2))                 # a j | b' be
    T2 = np.tensordot(T1, A, axes=([1, 3], [2, 3]))             # a b' | al i
    return np.ascontiguousarray(np.tensordot(x_bra, T2, axes=([1, 2], [3, 1])).transpose(0, 2, 1))


def enrich_right(x_k, z_k, x_k1, delta: float = 0.0, max_rank: int | None = None):
    """AMEn enrichment: [x_k | z_k] along the right bond, [x_{k+1}; 0], then one truncated SVD
    step moving the (trivial, l = 1) block index right -- x_k' left-orthonormal."""
    rl, n, rx = x_k.shape
    cat = np.concatenate([x_k, z_k], axis=2)
    cat1 = np.concatenate([x_k1, np.zeros((z_k.shape[2],) + x_k1.shape[1:])], axis=0)
    xk, x1 = block_move_right(cat.reshape(rl, n, 1, -1), cat1, delta, max_rank)
    return xk, x1[:, :, 0, :]
