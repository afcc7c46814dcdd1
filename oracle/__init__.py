"""ctypes binding of the plain C oracle (oracle/tt_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(paper_2509_11890_b200) never imports it, and this package imports nothing from there.
Arguments are numpy float64 arrays on the host; shapes follow SURVEY.md §8 Notation.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tt_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=c99", "-fPIC", "-shared"]
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with plain -O2 (no -ffast-math, no -march) into oracle/liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, dp, p = ctypes.c_int64, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p
        L.tt_oracle_local_matvec.argtypes = [i64] * 5 + [p] * 5
        L.tt_oracle_local_matvec_batched.argtypes = [i64] * 6 + [p] * 5
        L.tt_oracle_interface_left.argtypes = [i64] * 5 + [p] * 4
        L.tt_oracle_interface_right.argtypes = [i64] * 5 + [p] * 4
        L.tt_oracle_sweep_interfaces.argtypes = [i64, p, p, p, p, p, p, p, ctypes.c_int]
        L.tt_oracle_operator_apply.argtypes = [i64, p, p, p, p, p, p, p]
        L.tt_oracle_apply_core.argtypes = [i64] * 6 + [p] * 3
        L.tt_oracle_local_matvec_two_site.argtypes = [i64] * 7 + [p] * 6
        for f in ("tt_oracle_local_matvec", "tt_oracle_local_matvec_batched",
                  "tt_oracle_interface_left", "tt_oracle_interface_right",
                  "tt_oracle_sweep_interfaces", "tt_oracle_operator_apply",
                  "tt_oracle_apply_core", "tt_oracle_local_matvec_two_site"):
            getattr(L, f).restype = ctypes.c_int
        _ = dp
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _c(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(st):
    if st != 0:
        raise OracleError(f"oracle status {st}")


def local_matvec(phiL, A, phiR, x):
    phiL, A, phiR, x = map(_c, (phiL, A, phiR, x))
    rl, n, rr = x.shape
    Rl, Rr = A.shape[0], A.shape[3]
    y = np.empty_like(x)
    _check(lib().tt_oracle_local_matvec(rl, n, rr, Rl, Rr, _p(phiL), _p(A), _p(phiR), _p(x), _p(y)))
    return y


def local_matvec_batched(phiL, A, phiR, X):
    phiL, A, phiR, X = map(_c, (phiL, A, phiR, X))
    rl, n, nvec, rr = X.shape
    Rl, Rr = A.shape[0], A.shape[3]
    Y = np.empty_like(X)
    _check(lib().tt_oracle_local_matvec_batched(rl, n, rr, Rl, Rr, nvec, _p(phiL), _p(A),
                                                _p(phiR), _p(X), _p(Y)))
    return Y


def interface_left(phiL_prev, A, x):
    phiL_prev, A, x = map(_c, (phiL_prev, A, x))
    rl, n, rr = x.shape
    Rl, Rr = A.shape[0], A.shape[3]
    out = np.empty((rr, Rr, rr))
    _check(lib().tt_oracle_interface_left(rl, n, rr, Rl, Rr, _p(phiL_prev), _p(A), _p(x), _p(out)))
    return out


def interface_right(phiR_next, A, x):
    phiR_next, A, x = map(_c, (phiR_next, A, x))
    rl, n, rr = x.shape
    Rl, Rr = A.shape[0], A.shape[3]
    out = np.empty((rl, Rl, rl))
    _check(lib().tt_oracle_interface_right(rl, n, rr, Rl, Rr, _p(phiR_next), _p(A), _p(x), _p(out)))
    return out


def _ptr_array(arrs):
    return (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def sweep_interfaces(x_cores, A_cores, directions: int = 3):
    """Returns (phiL, phiR): lists of d+1 arrays, phiL[k]/phiR[k] of shape (r[k],R[k],r[k])."""
    x_cores = [_c(c) for c in x_cores]
    A_cores = [_c(c) for c in A_cores]
    d = len(x_cores)
    n = np.array([c.shape[1] for c in x_cores], dtype=np.int64)
    r = np.array([c.shape[0] for c in x_cores] + [x_cores[-1].shape[2]], dtype=np.int64)
    R = np.array([c.shape[0] for c in A_cores] + [A_cores[-1].shape[3]], dtype=np.int64)
    phiL = [np.zeros((r[k], R[k], r[k])) for k in range(d + 1)]
    phiR = [np.zeros((r[k], R[k], r[k])) for k in range(d + 1)]
    pl, pr = _ptr_array(phiL), _ptr_array(phiR)
    _check(lib().tt_oracle_sweep_interfaces(
        d, _p(n), _p(r), _p(R), _ptr_array(x_cores), _ptr_array(A_cores),
        pl if directions & 1 else None, pr if directions & 2 else None, directions))
    return phiL, phiR


def operator_apply(x_cores, A_cores):
    x_cores = [_c(c) for c in x_cores]
    A_cores = [_c(c) for c in A_cores]
    d = len(x_cores)
    n_row = np.array([c.shape[1] for c in A_cores], dtype=np.int64)
    n_col = np.array([c.shape[2] for c in A_cores], dtype=np.int64)
    r = np.array([c.shape[0] for c in x_cores] + [x_cores[-1].shape[2]], dtype=np.int64)
    R = np.array([c.shape[0] for c in A_cores] + [A_cores[-1].shape[3]], dtype=np.int64)
    z = [np.empty((r[k] * R[k], n_row[k], r[k + 1] * R[k + 1])) for k in range(d)]
    _check(lib().tt_oracle_operator_apply(d, _p(n_row), _p(n_col), _p(r), _p(R),
                                          _ptr_array(x_cores), _ptr_array(A_cores), _ptr_array(z)))
    return z


def apply_core(x, A):
    """One core of the unrounded apply: x (rl,nj,rr), A (Rl,ni,nj,Rr) -> (rl*Rl, ni, rr*Rr)."""
    x, A = _c(x), _c(A)
    rl, nj, rr = x.shape
    Rl, ni, _, Rr = A.shape
    z = np.empty((rl * Rl, ni, rr * Rr))
    _check(lib().tt_oracle_apply_core(rl, ni, nj, rr, Rl, Rr, _p(x), _p(A), _p(z)))
    return z


def local_matvec_two_site(phiL, A1, A2, phiR, w):
    """Two-site local matvec on a supercore w (rl, n1, n2, rr)."""
    phiL, A1, A2, phiR, w = map(_c, (phiL, A1, A2, phiR, w))
    rl, n1, n2, rr = w.shape
    Rl, Rm, Rr = A1.shape[0], A1.shape[3], A2.shape[3]
    y = np.empty_like(w)
    _check(lib().tt_oracle_local_matvec_two_site(rl, n1, n2, rr, Rl, Rm, Rr, _p(phiL), _p(A1),
                                                 _p(A2), _p(phiR), _p(w), _p(y)))
    return y


def block_local_matvec(ops, terms, X):
    """the projected KKT block system acting on a
    Block-TT core X (rl, n, nblocks, rr) whose block index is the KKT component:
        Y[:, :, row, :] = sum over terms (row, col, op, op2, coeff) of
                          coeff * L_op( L_op2( X[:, :, col, :] ) )   (op2 = -1: L_op only)
    where L_o is the projected operator of ops[o] = (phiL, A, phiR) (all sharing the frame).
    Plain loops over the terms; each L_o is tt_oracle_local_matvec."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    Y = np.zeros_like(X)
    for (row, col, op, op2, coeff) in terms:
        v = np.ascontiguousarray(X[:, :, col, :])
        if op2 >= 0:
            v = local_matvec(*ops[op2], v)
        Y[:, :, row, :] += coeff * local_matvec(*ops[op], v)
    return Y
