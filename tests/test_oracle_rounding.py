"""Pins for the orthonormalisation / TT-rounding oracle (oracle/rounding.py), CPU only."""
import numpy as np
import pytest

import ttgen
from dense_ref import full_vector, left_interface, rel_fro
from oracle.rounding import (core_lq_right, core_qr_left, orthonormalise_left,
                             orthonormalise_right, tt_round)


def _tt(seed, r, N=4):
    return ttgen.gaussian_tt_vector(np.random.default_rng(seed), N, r)


def _tt_sum(a, b):
    d = len(a)
    out = []
    for k in range(d):
        ca, cb = a[k], b[k]
        if k == 0:
            out.append(np.concatenate([ca, cb], axis=2))
        elif k == d - 1:
            out.append(np.concatenate([ca, cb], axis=0))
        else:
            c = np.zeros((ca.shape[0] + cb.shape[0], ca.shape[1], ca.shape[2] + cb.shape[2]))
            c[:ca.shape[0], :, :ca.shape[2]] = ca
            c[ca.shape[0]:, :, ca.shape[2]:] = cb
            out.append(c)
    return out


def test_core_qr_and_lq():
    rng = np.random.default_rng(1)
    c = rng.standard_normal((6, 4, 9))
    Q, R = core_qr_left(c)
    assert np.allclose(np.tensordot(Q, R, axes=(2, 0)), c, atol=1e-13)
    M = Q.reshape(24, 9)
    assert np.allclose(M.T @ M, np.eye(9), atol=1e-13)
    assert np.allclose(R, np.triu(R)) and (np.diag(R) >= 0).all()
    L, Q2 = core_lq_right(c)
    assert np.allclose(np.tensordot(L, Q2, axes=(1, 0)), c, atol=1e-13)
    M2 = Q2.reshape(6, 36)
    assert np.allclose(M2 @ M2.T, np.eye(6), atol=1e-13)
    assert np.allclose(L, np.tril(L))


def test_orthonormalise_preserves_tensor_and_gauge():
    x = _tt(2, [1, 4, 8, 8, 4, 1])
    v = full_vector(x)
    xl = orthonormalise_left(x)
    assert rel_fro(full_vector(xl), v) < 1e-13
    for k in range(1, 5):
        L = left_interface(xl, k)
        assert np.allclose(L.T @ L, np.eye(L.shape[1]), atol=1e-13)
    xr = orthonormalise_right(x)
    assert rel_fro(full_vector(xr), v) < 1e-13


def test_round_error_bound_and_exact_case():
    """||T - round(T, delta)|| <= delta ||T|| (Oseledets Thm. 2.2 via Alg. 2), and rounding
    the formal sum T + T (ranks doubled) at delta ~ 0 recovers ranks <= those of T."""
    x = _tt(3, [1, 4, 10, 12, 6, 1])
    v = full_vector(x)
    for delta in (1e-1, 1e-2, 1e-4):
        y = tt_round(x, delta)
        assert rel_fro(full_vector(y), v) <= delta * (1 + 1e-12)
    xx = _tt_sum(x, x)
    y = tt_round(xx, 1e-12)
    assert rel_fro(full_vector(y), 2 * v) < 1e-11
    for k in range(len(x)):
        assert y[k].shape[2] <= x[k].shape[2]


def test_round_rank_one_stays_rank_one():
    """The identity / all-ones TT vectors are rank 1."""
    ones = [np.ones((1, 4, 1)) for _ in range(5)]
    y = tt_round(_tt_sum(ones, ones), 1e-12)
    assert all(c.shape[0] == 1 and c.shape[2] == 1 for c in y)
    assert rel_fro(full_vector(y), 2 * full_vector(ones)) < 1e-13
