"""Pins for the Petrov-Galerkin / AMEn-enrichment oracle (oracle/petrov.py), CPU only: dense
two-train frames, the square case of the C oracle, and the
invariance of the represented tensor under enrichment."""
import numpy as np

import oracle
import ttgen
from dense_ref import frame, full_matrix, full_vector, rel_fro
from oracle.petrov import enrich_right, interface_left_pg, interface_right_pg, local_matvec_pg


def _trains(seed=61, d=5, N=4, rx=3, rz=2, R=3):
    rng = np.random.default_rng(seed)
    x = ttgen.gaussian_tt_vector(rng, N, ttgen.capped_ranks(d, N, rx))
    z = ttgen.gaussian_tt_vector(rng, N, ttgen.capped_ranks(d, N, rz))
    A = ttgen.gaussian_tt_matrix(rng, N, N, ttgen.capped_ranks(d, N * N, R))
    return rng, x, z, A


def _interfaces(z, A, x):
    """Two-train interfaces by chaining the oracle's own updates (both directions)."""
    d = len(x)
    pl = [np.ones((1, 1, 1))]
    for k in range(d - 1):
        pl.append(interface_left_pg(pl[-1], A[k], z[k], x[k]))
    pr = [np.ones((1, 1, 1))]
    for k in range(d - 1, 0, -1):
        pr.insert(0, interface_right_pg(pr[0], A[k], z[k], x[k]))
    return pl, [None] + pr


def test_pg_matvec_is_two_train_projection():
    """Z_{!=k}^T A X_{!=k} vec(x_k) from dense frames of two different trains."""
    rng, x, z, A = _trains()
    pl, pr = _interfaces(z, A, x)
    Af = full_matrix(A)
    for k in range(len(x)):
        ref = frame(z, k).T @ Af @ frame(x, k) @ x[k].ravel()
        got = local_matvec_pg(pl[k], A[k], pr[k + 1], x[k])
        assert rel_fro(got.ravel(), ref) <= 1e-12


def test_pg_interfaces_close_to_bilinear_form():
    """phiL after all cores = phiR before all cores = z^T A x (dense)."""
    rng, x, z, A = _trains(62)
    pl, pr = _interfaces(z, A, x)
    d = len(x)
    full = interface_left_pg(pl[d - 1], A[d - 1], z[d - 1], x[d - 1])
    ref = full_vector(z) @ full_matrix(A) @ full_vector(x)
    assert abs(full.item() - ref) <= 1e-12 * abs(ref)
    first = interface_right_pg(pr[1], A[0], z[0], x[0])
    assert abs(first.item() - ref) <= 1e-12 * abs(ref)


def test_pg_square_case_is_the_c_oracle():
    rng, x, z, A = _trains(63)
    k = 2
    pl, pr = oracle.sweep_interfaces(x, A, 3)
    a = local_matvec_pg(pl[k], A[k], pr[k + 1], x[k])
    b = oracle.local_matvec(pl[k], A[k], pr[k + 1], x[k])
    assert rel_fro(a, b) <= 1e-13
    X = rng.standard_normal(x[k].shape[:2] + (3,) + x[k].shape[2:])
    assert rel_fro(local_matvec_pg(pl[k], A[k], pr[k + 1], X),
                   oracle.local_matvec_batched(pl[k], A[k], pr[k + 1], X)) <= 1e-13
    assert rel_fro(interface_left_pg(pl[k], A[k], x[k], x[k]),
                   oracle.interface_left(pl[k], A[k], x[k])) <= 1e-13
    assert rel_fro(interface_right_pg(pr[k + 1], A[k], x[k], x[k]),
                   oracle.interface_right(pr[k + 1], A[k], x[k])) <= 1e-13


def test_projected_rhs_identity_operator():
    """X_{!=k}^T vec(B): identity operator cores, B as ket."""
    rng = np.random.default_rng(64)
    d, N = 4, 4
    x = ttgen.gaussian_tt_vector(rng, N, [1, 3, 5, 3, 1])
    B = ttgen.gaussian_tt_vector(rng, N, [1, 2, 4, 2, 1])
    I = ttgen.identity_operator(d, N)
    pl, pr = _interfaces(x, I, B)
    for k in range(d):
        ref = frame(x, k).T @ full_vector(B)
        assert rel_fro(local_matvec_pg(pl[k], I[k], pr[k + 1], B[k]).ravel(), ref) <= 1e-12


def test_enrichment_keeps_tensor_and_spans_residual():
    rng = np.random.default_rng(65)
    x = ttgen.gaussian_tt_vector(rng, 4, [1, 4, 6, 4, 1])
    k = 1
    zk = rng.standard_normal((4, 4, 3))
    xk, x1 = enrich_right(x[k], zk, x[k + 1])
    assert xk.shape == (4, 4, 9) and x1.shape == (9, 4, 4)
    M = xk.reshape(16, 9)
    assert np.allclose(M.T @ M, np.eye(9), atol=1e-13)
    y = x[:k] + [xk, x1] + x[k + 2:]
    assert rel_fro(full_vector(y), full_vector(x)) <= 1e-13
    # the enriched core spans both x_k and the residual core
    P = M @ M.T
    for c in (x[k].reshape(16, -1), zk.reshape(16, -1)):
        assert np.abs(P @ c - c).max() <= 1e-12 * np.abs(c).max()
