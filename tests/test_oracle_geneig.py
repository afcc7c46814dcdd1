"""Pins for the step-length eigenproblem oracle (oracle/geneig.py), CPU only.

Each pin checks the oracle against something other than itself: the frame-matrix projection
of dense_ref, closed-form spectra of Kronecker sums, and the defining
property of the step length (X + alpha dX singular at alpha = 1/lam_max).
"""
import numpy as np
import pytest

import oracle
import ttgen
from dense_ref import full_matrix, projected_operator
from oracle.geneig import (block_columns, columns_block, geneig_dense, local_geneig,
                           local_operator_dense, step_length)


def mixed_frame(x, k, two_site=False):
    """Mixed-canonical train: left-orthonormal cores < k, right-orthonormal cores > k (> k+1
    for the two-site frame)."""
    xl, xr = ttgen.left_orthonormalise(x), ttgen.right_orthonormalise(x)
    last = k + 1 if two_site else k
    return xl[:k] + [x[j] for j in range(k, last + 1)] + xr[last + 1:]


def kron_sum_tt(F_list):
    """TT matrix of sum_k I (x) .. F_k .. (x) I (rank 2): cores [F I], [[I 0],[F I]], [[I],[F]]."""
    d = len(F_list)
    n = F_list[0].shape[0]
    I = np.eye(n)
    cores = []
    for k, F in enumerate(F_list):
        if d == 1:
            cores.append(F.reshape(1, n, n, 1))
        elif k == 0:
            c = np.zeros((1, n, n, 2))
            c[0, :, :, 0], c[0, :, :, 1] = F, I
            cores.append(c)
        elif k == d - 1:
            c = np.zeros((2, n, n, 1))
            c[0, :, :, 0], c[1, :, :, 0] = I, F
            cores.append(c)
        else:
            c = np.zeros((2, n, n, 2))
            c[0, :, :, 0], c[1, :, :, 0], c[1, :, :, 1] = I, F, I
            cores.append(c)
    return cores


def local_ops(x, ops, k):
    pl_pr = [oracle.sweep_interfaces(x, A, 3) for A in ops]
    return [(pl[k], A[k], pr[k + 1]) for (pl, pr), A in zip(pl_pr, ops)]


def test_local_operator_dense_is_projected_operator():
    """(M) as a matrix equals X_{!=k}^T A X_{!=k} built from the dense frame."""
    rng = np.random.default_rng(41)
    d, n = 5, 2
    x = ttgen.gaussian_tt_vector(rng, n, ttgen.capped_ranks(d, n, 3))
    A = ttgen.symmetric_tt_matrix(rng, d, n, 3)
    for k in (0, 2, 4):
        mixed = mixed_frame(x, k)
        (op,) = local_ops(mixed, [A], k)
        ref = projected_operator(mixed, full_matrix(A), k)
        got = local_operator_dense(*op)
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


def test_kron_sum_spectrum_closed_form():
    """Full-rank orthonormal frame: the local operator is orthogonally similar to A, whose
    Kronecker-sum spectrum is {f_i1 + ... + f_id} (closed form)."""
    rng = np.random.default_rng(42)
    d, n = 4, 2
    f = np.array([-0.7, 1.9])
    Q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    F = Q @ np.diag(f) @ Q.T
    A = kron_sum_tt([F] * d)
    x = ttgen.gaussian_tt_vector(rng, n, [1, 2, 4, 2, 1])
    k = 2
    mixed = mixed_frame(x, k)
    (op,) = local_ops(mixed, [A], k)
    sums = sorted((sum(c) for c in np.array(np.meshgrid(*[f] * d)).reshape(d, -1).T), reverse=True)
    lam, V = local_geneig(op, None, 6)
    assert np.allclose(lam, sums[:6], rtol=0, atol=1e-12)
    assert np.allclose(V.T @ V, np.eye(6), atol=1e-12)


def test_generalised_kron_sum_closed_form():
    """A = sum F_k, B = sum G_k with F, G sharing eigenvectors: the pencil eigenvalues are
    (f_i1 + .. + f_id) / (g_i1 + .. + g_id)."""
    rng = np.random.default_rng(43)
    d, n = 4, 2
    f, g = np.array([0.3, -1.1]), np.array([0.5, 2.0])
    Q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    A = kron_sum_tt([Q @ np.diag(f) @ Q.T] * d)
    B = kron_sum_tt([Q @ np.diag(g) @ Q.T] * d)
    x = ttgen.gaussian_tt_vector(rng, n, [1, 2, 4, 2, 1])
    k = 1
    mixed = mixed_frame(x, k)
    opA, opB = local_ops(mixed, [A, B], k)
    idx = np.array(np.meshgrid(*[[0, 1]] * d)).reshape(d, -1).T
    ratios = sorted((f[i].sum() / g[i].sum() for i in idx), reverse=True)
    lam, V = local_geneig(opA, opB, 5)
    assert np.allclose(lam, ratios[:5], rtol=0, atol=1e-12)
    LB = local_operator_dense(*opB)
    assert np.allclose(V.T @ LB @ V, np.eye(5), atol=1e-11)


def test_geneig_reduces_to_nonsymmetric_eig():
    """Random SPD pencil: the eigenvalues equal those of B^{-1} A from the general
    (nonsymmetric) eigensolver."""
    rng = np.random.default_rng(44)
    m = 30
    A = rng.standard_normal((m, m))
    A = A + A.T
    G = rng.standard_normal((m, m))
    B = G @ G.T + m * np.eye(m)
    lam, V = geneig_dense(A, B, 7)
    ev = np.sort(np.linalg.eigvals(np.linalg.solve(B, A)).real)[::-1]
    assert np.allclose(lam, ev[:7], rtol=0, atol=1e-10)
    assert np.abs(A @ V - B @ V * lam).max() <= 1e-10 * np.abs(A).max()


def test_step_length_makes_x_singular():
    """Full frame (local = global pencil): alpha = step_length(lam_max(-dX, X)) is the
    largest step keeping X + alpha dX positive semidefinite."""
    rng = np.random.default_rng(45)
    d, n = 4, 2
    X = ttgen.spd_factor(rng, d, n, 3)
    dX = ttgen.symmetric_tt_matrix(rng, d, n, 3, fro=12.0)
    negdX = [c.copy() for c in dX]
    negdX[0] = -negdX[0]
    x = ttgen.gaussian_tt_vector(rng, n, [1, 2, 4, 2, 1])
    k = 2
    mixed = mixed_frame(x, k)
    opA, opB = local_ops(mixed, [negdX, X], k)
    lam, _ = local_geneig(opA, opB, 1)
    alpha = step_length(lam[0])
    Xf, dXf = full_matrix(X), full_matrix(dX)
    assert 0.0 < alpha < 1.0, "the fixture must produce a step below the cap"
    assert abs(np.linalg.eigvalsh(Xf + alpha * dXf)[0]) <= 1e-10 * np.abs(Xf).max()
    assert np.linalg.eigvalsh(Xf + 0.999 * alpha * dXf)[0] > 0.0
    assert np.linalg.eigvalsh(Xf + 1.001 * alpha * dXf)[0] < 0.0


def test_step_length_cap():
    assert step_length(0.25) == 1.0 and step_length(-3.0) == 1.0 and step_length(0.0) == 1.0
    assert step_length(4.0) == 0.25


def test_block_column_layout_roundtrip():
    rng = np.random.default_rng(46)
    X = rng.standard_normal((3, 4, 5, 2))
    V = block_columns(X)
    assert V.shape == (24, 5)
    for j in range(5):
        assert np.array_equal(V[:, j], X[:, :, j, :].ravel())
    assert np.array_equal(columns_block(V, 3, 4, 2), X)
