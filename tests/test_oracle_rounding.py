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


# --------------------------------------------------------------------------------------
# block-index move: one SVD step of TT rounding
# --------------------------------------------------------------------------------------
from oracle.rounding import block_move_left, block_move_right  # noqa: E402


def _pair_right(Wk_hat, Wk1):
    """Block tensors of the pair: T[a, i, l, j, c] = sum_b Wk_hat[a,i,l,b] Wk1[b,j,c]."""
    return np.einsum("ailb,bjc->ailjc", Wk_hat, Wk1)


def _pair_after_right(Wk, Wk1_hat):
    return np.einsum("ais,sjlc->ailjc", Wk, Wk1_hat)


def _graded(rng, m, q, sig):
    """m x q matrix with prescribed singular values (random orthonormal factors)."""
    U = np.linalg.qr(rng.standard_normal((m, len(sig))))[0]
    V = np.linalg.qr(rng.standard_normal((q, len(sig))))[0]
    return (U * sig) @ V.T


def test_block_move_right_exact_and_orthonormal():
    rng = np.random.default_rng(21)
    Wk_hat = rng.standard_normal((3, 4, 4, 5))
    Wk1 = rng.standard_normal((5, 4, 2))
    Wk, W1 = block_move_right(Wk_hat, Wk1)
    assert Wk.shape == (3, 4, 12) and W1.shape == (12, 4, 4, 2)
    M = Wk.reshape(12, 12)
    assert np.allclose(M.T @ M, np.eye(12), atol=1e-13)
    T0, T1 = _pair_right(Wk_hat, Wk1), _pair_after_right(Wk, W1)
    assert rel_fro(T1, T0) <= 1e-13


def test_block_move_truncation_is_eckart_young():
    """With Wk1 right-orthonormal the pair's error equals the discarded singular values
    (Eckart-Young), is <= delta, and one rank fewer would exceed delta."""
    rng = np.random.default_rng(22)
    r0, n0, l, r1 = 4, 4, 4, 6
    sig = np.array([3.0, 2.0, 1.0, 0.5, 1e-3, 5e-4, 1e-5, 1e-6])
    Wk_hat = _graded(rng, r0 * n0, l * r1, sig).reshape(r0, n0, l, r1)
    Q = np.linalg.qr(rng.standard_normal((4 * 3, r1)))[0]        # (n1 r2) x r1, orthonormal
    Wk1 = Q.T.reshape(r1, 4, 3)
    T0 = _pair_right(Wk_hat, Wk1)
    for delta, s_exp in ((1e-2, 4), (1e-4, 6), (1e-6, 7)):
        Wk, W1 = block_move_right(Wk_hat, Wk1, delta)
        assert Wk.shape[2] == s_exp
        err = np.linalg.norm(_pair_after_right(Wk, W1) - T0)
        tail = np.linalg.norm(sig[s_exp:])
        assert abs(err - tail) <= 1e-12 * np.linalg.norm(sig)
        assert err <= delta * np.linalg.norm(sig) + 1e-14
        if s_exp > 1:
            assert np.linalg.norm(sig[s_exp - 1:]) > delta * np.linalg.norm(sig)
    Wk, W1 = block_move_right(Wk_hat, Wk1, 0.0, max_rank=3)
    assert Wk.shape[2] == 3


def test_block_move_left_exact_and_orthonormal():
    rng = np.random.default_rng(23)
    Wkm1 = rng.standard_normal((2, 4, 5))
    Wk_hat = rng.standard_normal((5, 4, 3, 6))
    Wh, Wk = block_move_left(Wkm1, Wk_hat)
    s = Wk.shape[0]
    assert s == min(5 * 3, 4 * 6) and Wh.shape == (2, 4, 3, s)
    R = Wk.reshape(s, 24)
    assert np.allclose(R @ R.T, np.eye(s), atol=1e-13)
    T0 = np.einsum("ajb,bilc->ajilc", Wkm1, Wk_hat)
    T1 = np.einsum("ajls,sic->ajilc", Wh, Wk)
    assert rel_fro(T1, T0) <= 1e-13


def test_block_move_round_trip():
    """Moving right then back left reproduces the block tensors (delta = 0)."""
    rng = np.random.default_rng(24)
    Wk_hat = rng.standard_normal((3, 4, 2, 5))
    Wk1 = rng.standard_normal((5, 4, 3))
    Wk, W1 = block_move_right(Wk_hat, Wk1)
    Wh, Wk1b = block_move_left(Wk, W1)
    T0 = _pair_right(Wk_hat, Wk1)
    T2 = np.einsum("ails,sjc->ailjc", Wh, Wk1b)
    assert rel_fro(T2, T0) <= 1e-12
