"""Pins for the GMRES oracle (oracle/gmres.py) against dense linear algebra (CPU only)."""
import numpy as np
import pytest

import oracle
import ttgen
from dense_ref import full_matrix, projected_operator
from oracle.gmres import gmres, local_gmres_batched


def test_finite_termination_dense():
    """Unrestarted GMRES on an n x n system terminates with the exact solution in n steps
    (Saad Prop. 6.10); checked against numpy.linalg.solve on a nonsymmetric matrix."""
    rng = np.random.default_rng(1)
    n = 40
    M = rng.standard_normal((n, n)) + 8 * np.eye(n)
    f = rng.standard_normal(n)
    x, rel, its = gmres(lambda v: M @ v, f, np.zeros(n), m=n, cycles=1, tol=1e-15)
    ref = np.linalg.solve(M, f)
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) < 1e-12
    assert its <= n


def test_residual_estimate_is_true_residual():
    rng = np.random.default_rng(2)
    n = 30
    M = rng.standard_normal((n, n)) + 6 * np.eye(n)
    f = rng.standard_normal(n)
    for m in (3, 7, 12):
        x, rel, _ = gmres(lambda v: M @ v, f, np.zeros(n), m=m, cycles=1, tol=0.0)
        true = np.linalg.norm(f - M @ x) / np.linalg.norm(f)
        assert abs(true - rel) <= 1e-10


def test_residual_monotone_in_m():
    """GMRES minimises the residual over nested Krylov spaces: non-increasing in m."""
    rng = np.random.default_rng(3)
    n = 25
    M = rng.standard_normal((n, n)) + 5 * np.eye(n)
    f = rng.standard_normal(n)
    prev = np.inf
    for m in range(1, 15):
        _, rel, _ = gmres(lambda v: M @ v, f, np.zeros(n), m=m, cycles=1, tol=0.0)
        assert rel <= prev + 1e-14
        prev = rel


def test_identity_one_step():
    f = np.arange(1.0, 9.0)
    x, rel, its = gmres(lambda v: v, f, np.zeros(8), m=5, cycles=2, tol=1e-14)
    assert its == 1 and np.allclose(x, f, rtol=0, atol=1e-14)


def _spd_local_system(seed=5, d=4):
    """A config-2-like local system: Kronecker-sum SPD operator (readings R1-R4), mixed
    canonical frame (left-orthonormal cores left of k, right-orthonormal right of k)."""
    n = 2
    N = n * n
    rng = np.random.default_rng(seed)
    Xf = ttgen.spd_factor(rng, d, n, 2)
    Zf = ttgen.spd_factor(rng, d, n, 2)
    A = ttgen.kron_sum_operator(Xf, Zf, n)
    r = ttgen.capped_ranks(d, N, 6)
    x = ttgen.gaussian_tt_vector(rng, N, r)
    xl, xr = ttgen.left_orthonormalise(x), ttgen.right_orthonormalise(x)
    k = 2
    mixed = xl[:k] + [x[k]] + xr[k + 1:]
    pl, _ = oracle.sweep_interfaces(mixed, A, 1)
    _, pr = oracle.sweep_interfaces(mixed, A, 2)
    return mixed, A, k, pl[k], pr[k + 1], rng


def test_local_gmres_matches_dense_solve():
    """Converged matrix-free GMRES on the projected operator equals the dense
    solve of X_{!=k}^T A X_{!=k} y = f built from the frame matrix."""
    mixed, A, k, phiL, phiR, rng = _spd_local_system()
    shape = mixed[k].shape
    Ldense = projected_operator(mixed, full_matrix(A), k)
    K = 3
    F = rng.standard_normal((shape[0], shape[1], K, shape[2]))
    X, rel, its = local_gmres_batched(phiL, A[k], phiR, F, np.zeros_like(F), m=20, cycles=5,
                                      tol=1e-14)
    for j in range(K):
        ref = np.linalg.solve(Ldense, F[:, :, j, :].ravel())
        got = X[:, :, j, :].ravel()
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-12
    assert (rel <= 1e-14).all()


def test_local_gmres_restarts_converge_spd():
    """Restarted GMRES(4) on the SPD local operator: Poincare separation bounds its spectrum
    by A's, so the restarts converge."""
    mixed, A, k, phiL, phiR, rng = _spd_local_system(seed=7)
    shape = mixed[k].shape
    F = rng.standard_normal((shape[0], shape[1], 2, shape[2]))
    X, rel, its = local_gmres_batched(phiL, A[k], phiR, F, np.zeros_like(F), m=4, cycles=60,
                                      tol=1e-12)
    assert (rel <= 1e-12).all()
    Ldense = projected_operator(mixed, full_matrix(A), k)
    for j in range(2):
        res = F[:, :, j, :].ravel() - Ldense @ X[:, :, j, :].ravel()
        assert np.linalg.norm(res) / np.linalg.norm(F[:, :, j, :]) < 1e-11


def test_zero_rhs():
    x, rel, its = gmres(lambda v: 2 * v, np.zeros(5), np.ones(5), m=3, cycles=2, tol=1e-12)
    assert not x.any() and rel == 0.0 and its == 0


# --------------------------------------------------------------------------------------
# accelerated GMRES (LGMRES, Baker et al. 2005) — PAPER.md:488 "accelerated GMRES"
# --------------------------------------------------------------------------------------
def test_lgmres_first_cycle_is_gmres():
    rng = np.random.default_rng(11)
    n = 30
    M = rng.standard_normal((n, n)) + 6 * np.eye(n)
    f = rng.standard_normal(n)
    a = gmres(lambda v: M @ v, f, np.zeros(n), m=6, cycles=1, tol=0.0, k=0)
    b = gmres(lambda v: M @ v, f, np.zeros(n), m=6, cycles=1, tol=0.0, k=2)
    assert np.array_equal(a[0], b[0]) and a[2] == b[2]


def test_lgmres_cycle_minimises_over_augmented_space():
    """The second cycle's iterate minimises ||f - M x|| over x1 + span(K_m(M, r1) + z1) with
    z1 = x1 - x0 (dense least squares on an explicit basis)."""
    rng = np.random.default_rng(12)
    n, m = 40, 5
    M = rng.standard_normal((n, n)) + 7 * np.eye(n)
    f = rng.standard_normal(n)
    x0 = np.zeros(n)
    x1, _, _ = gmres(lambda v: M @ v, f, x0, m=m, cycles=1, tol=0.0, k=1)
    x2, rel2, _ = gmres(lambda v: M @ v, f, x0, m=m, cycles=2, tol=0.0, k=1)
    r1 = f - M @ x1
    K = [r1]
    for _ in range(m - 1):
        K.append(M @ K[-1])
    W = np.linalg.qr(np.column_stack(K + [x1 - x0]))[0]
    y = np.linalg.lstsq(M @ W, r1, rcond=None)[0]
    best = np.linalg.norm(r1 - M @ W @ y)
    got = np.linalg.norm(f - M @ x2)
    assert abs(got - best) <= 1e-10 * np.linalg.norm(f)
    assert abs(rel2 - got / np.linalg.norm(f)) <= 1e-10


def test_lgmres_converges_to_dense_solve():
    mixed, A, k, phiL, phiR, rng = _spd_local_system(seed=13)
    shape = mixed[k].shape
    F = rng.standard_normal((shape[0], shape[1], 2, shape[2]))
    X, rel, its = local_gmres_batched(phiL, A[k], phiR, F, np.zeros_like(F), m=4, cycles=60,
                                      tol=1e-12, k=2)
    assert (rel <= 1e-12).all()
    Ldense = projected_operator(mixed, full_matrix(A), k)
    for j in range(2):
        ref = np.linalg.solve(Ldense, F[:, :, j, :].ravel())
        assert np.linalg.norm(X[:, :, j, :].ravel() - ref) / np.linalg.norm(ref) < 1e-10
