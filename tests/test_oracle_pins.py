"""Pins for the CPU oracle against things other than itself (CPU only, -m "not gpu").

Each test cites the passage that fixes the expected value.  The dense side (dense_ref.py)
materialises the full objects from the paper's definitions; the oracle never does.
"""
import json
import os

import numpy as np
import pytest

import oracle
import ttgen
from dense_ref import (frame, full_matrix, full_vector, phiL_dense, phiR_dense,
                       projected_operator, rel_fro, unvec_tt_dense, vec_tt_dense)

TOL_DENSE = 1e-12   # brute force vs oracle, O(1)-scaled inputs, FP64 (DESIGN.md §3 A9)
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand_tt(seed, d, N, r, R, nvec=0):
    rng = np.random.default_rng(seed)
    x = ttgen.gaussian_tt_vector(rng, N, r)
    A = ttgen.gaussian_tt_matrix(rng, N, N, R)
    X = ttgen.random_block(rng, N, r, nvec) if nvec else None
    return x, A, X


SMALL_CASES = [
    # (seed, d, N, r, R)
    (11, 3, 4, [1, 3, 5, 1], [1, 2, 3, 1]),
    (12, 4, 4, [1, 8, 8, 8, 1], [1, 4, 4, 4, 1]),      # config-1 shape
    (13, 4, 3, [1, 2, 4, 3, 1], [1, 5, 1, 2, 1]),      # odd mode, rank-1 operator bond
    (14, 5, 2, [1, 2, 4, 4, 2, 1], [1, 3, 3, 3, 3, 1]),
    (15, 1, 5, [1, 1], [1, 1]),                         # d = 1: no interfaces
]


# --------------------------------------------------------------------------------------
# dense-reference self-checks (frame identity) — PAPER.md:257-263 Remark
# --------------------------------------------------------------------------------------
@pytest.mark.parametrize("case", SMALL_CASES)
def test_frame_identity(case):
    seed, d, N, r, R = case
    x, _, _ = _rand_tt(seed, d, N, r, R)
    v = full_vector(x)
    for k in range(d):
        assert rel_fro(frame(x, k) @ x[k].reshape(-1), v) < 1e-13


# --------------------------------------------------------------------------------------
# (M) local matvec == X_{!=k}^T A X_{!=k} vec(x_k)  — PAPER.md:289-292
# --------------------------------------------------------------------------------------
@pytest.mark.parametrize("case", SMALL_CASES)
def test_local_matvec_projected_operator(case):
    seed, d, N, r, R = case
    x, A, _ = _rand_tt(seed, d, N, r, R)
    Af = full_matrix(A)
    phiL, phiR = oracle.sweep_interfaces(x, A)
    for k in range(d):
        y = oracle.local_matvec(phiL[k], A[k], phiR[k + 1], x[k])
        ref = projected_operator(x, Af, k) @ x[k].reshape(-1)
        assert rel_fro(y.reshape(-1), ref) < TOL_DENSE, k


@pytest.mark.parametrize("case", SMALL_CASES)
def test_local_matvec_arbitrary_core(case):
    """The local operator applied to a core that is NOT x_k (GMRES iterate)."""
    seed, d, N, r, R = case
    x, A, _ = _rand_tt(seed, d, N, r, R)
    Af = full_matrix(A)
    phiL, phiR = oracle.sweep_interfaces(x, A)
    rng = np.random.default_rng(seed + 100)
    for k in range(d):
        v = rng.standard_normal(x[k].shape)
        y = oracle.local_matvec(phiL[k], A[k], phiR[k + 1], v)
        ref = projected_operator(x, Af, k) @ v.reshape(-1)
        assert rel_fro(y.reshape(-1), ref) < TOL_DENSE


# --------------------------------------------------------------------------------------
# (IL)/(IR) interfaces == dense partial products — PAPER.md:244-253
# --------------------------------------------------------------------------------------
@pytest.mark.parametrize("case", SMALL_CASES)
def test_interfaces_brute_force(case):
    seed, d, N, r, R = case
    x, A, _ = _rand_tt(seed, d, N, r, R)
    phiL, phiR = oracle.sweep_interfaces(x, A)
    for k in range(d + 1):
        assert rel_fro(phiL[k], phiL_dense(x, A, k)) < TOL_DENSE, ("L", k)
        assert rel_fro(phiR[k], phiR_dense(x, A, k)) < TOL_DENSE, ("R", k)


@pytest.mark.parametrize("case", SMALL_CASES)
def test_energy_identity_and_closure(case):
    """Restricted energy equals the full energy for every k:
    <x_k, y_k> = x^T A x = phiL[d] = phiR[0]."""
    seed, d, N, r, R = case
    x, A, _ = _rand_tt(seed, d, N, r, R)
    v = full_vector(x)
    e = v @ full_matrix(A) @ v
    phiL, phiR = oracle.sweep_interfaces(x, A)
    assert abs(phiL[d].item() - e) <= 1e-12 * max(1.0, abs(e))
    assert abs(phiR[0].item() - e) <= 1e-12 * max(1.0, abs(e))
    for k in range(d):
        y = oracle.local_matvec(phiL[k], A[k], phiR[k + 1], x[k])
        assert abs(np.vdot(x[k], y) - e) <= 1e-12 * max(1.0, abs(e))


def test_sweep_directions_and_single_calls():
    """H7 chaining == individual (IL)/(IR) calls; directions 1/2 fill only their side."""
    x, A, _ = _rand_tt(21, 4, 4, [1, 4, 6, 4, 1], [1, 3, 3, 3, 1])
    pl, pr = oracle.sweep_interfaces(x, A, 3)
    cur = np.ones((1, 1, 1))
    for k in range(4):
        cur = oracle.interface_left(cur, A[k], x[k])
        assert np.array_equal(cur, pl[k + 1])
    cur = np.ones((1, 1, 1))
    for k in range(3, -1, -1):
        cur = oracle.interface_right(cur, A[k], x[k])
        assert np.array_equal(cur, pr[k])
    pl1, pr1 = oracle.sweep_interfaces(x, A, 1)
    assert all(np.array_equal(a, b) for a, b in zip(pl1, pl))
    assert all(not p.any() for p in pr1)
    pl2, pr2 = oracle.sweep_interfaces(x, A, 2)
    assert all(not p.any() for p in pl2)
    assert all(np.array_equal(a, b) for a, b in zip(pr2, pr))


# --------------------------------------------------------------------------------------
# invariants: identity operator, orthonormal cores, linearity, symmetry
# --------------------------------------------------------------------------------------
def test_identity_operator_returns_x():
    """A = I (TT ranks 1) with identity interfaces -> y = x."""
    rng = np.random.default_rng(5)
    for (rl, n, rr) in [(1, 4, 1), (3, 4, 5), (8, 4, 8), (2, 7, 3)]:
        x = rng.standard_normal((rl, n, rr))
        phiL = np.eye(rl).reshape(rl, 1, rl)
        phiR = np.eye(rr).reshape(rr, 1, rr)
        y = oracle.local_matvec(phiL, np.eye(n).reshape(1, n, n, 1), phiR, x)
        assert np.array_equal(y, x)
        X = rng.standard_normal((rl, n, 3, rr))
        Y = oracle.local_matvec_batched(phiL, np.eye(n).reshape(1, n, n, 1), phiR, X)
        assert np.array_equal(Y, X)


@pytest.mark.parametrize("idx", [2, 3])
def test_orthonormal_cores_give_identity_interfaces(idx):
    """Left-orthonormal cores + identity operator -> phiL_k = I (SPEC.md:50
    'Gram matrix = identity to 1e-12'), right analogue with the LQ copy; full config scale."""
    inp = ttgen.make_inputs(idx)
    d, N = inp.cfg.d, inp.cfg.N
    I = ttgen.identity_operator(d, N)
    pl, _ = oracle.sweep_interfaces(inp.x, I, 1)
    for k in range(1, d):
        rk = pl[k].shape[0]
        assert np.abs(pl[k][:, 0, :] - np.eye(rk)).max() < 1e-12, k
    _, pr = oracle.sweep_interfaces(inp.x_right, I, 2)
    for k in range(1, d):
        rk = pr[k].shape[0]
        assert np.abs(pr[k][:, 0, :] - np.eye(rk)).max() < 1e-12, k
    # whole-vector norms are 1 (last / first core normalised), PAPER.md:252 boundary values
    assert abs(pl[d].item() - 1.0) < 1e-12 and abs(pr[0].item() - 1.0) < 1e-12


def test_linearity():
    x, A, _ = _rand_tt(31, 3, 4, [1, 4, 5, 1], [1, 3, 2, 1])
    pl, pr = oracle.sweep_interfaces(x, A)
    rng = np.random.default_rng(32)
    k = 1
    u = rng.standard_normal(x[k].shape)
    v = rng.standard_normal(x[k].shape)
    a, b = 1.7, -0.3
    f = lambda t: oracle.local_matvec(pl[k], A[k], pr[k + 1], t)
    assert rel_fro(f(a * u + b * v), a * f(u) + b * f(v)) < 1e-14
    # linear in A_k, phiL, phiR
    A2 = rng.standard_normal(A[k].shape)
    g = lambda Ak: oracle.local_matvec(pl[k], Ak, pr[k + 1], u)
    assert rel_fro(g(A[k] + 2 * A2), g(A[k]) + 2 * g(A2)) < 1e-14
    P2 = rng.standard_normal(pl[k].shape)
    h = lambda P: oracle.local_matvec(P, A[k], pr[k + 1], u)
    assert rel_fro(h(pl[k] - P2), h(pl[k]) - h(P2)) < 1e-14
    Q2 = rng.standard_normal(pr[k + 1].shape)
    q = lambda P: oracle.local_matvec(pl[k], A[k], P, u)
    assert rel_fro(q(pr[k + 1] + Q2), q(pr[k + 1]) + q(Q2)) < 1e-14


def test_symmetry_bra_ket():
    """Core-wise symmetric operator (A_k[.,i,j,.] = A_k[.,j,i,.]) + symmetric incoming Phi ->
    outgoing Phi symmetric under bra <-> ket; local operator symmetric."""
    rng = np.random.default_rng(41)
    x, A, _ = _rand_tt(42, 4, 4, [1, 4, 6, 5, 1], [1, 3, 3, 3, 1])
    A = [(c + c.transpose(0, 2, 1, 3)) / 2 for c in A]
    pl, pr = oracle.sweep_interfaces(x, A)
    for P in pl + pr:
        assert np.abs(P - P.transpose(2, 1, 0)).max() <= 1e-14 * max(1.0, np.abs(P).max())
    k = 2
    u = rng.standard_normal(x[k].shape)
    v = rng.standard_normal(x[k].shape)
    f = lambda t: oracle.local_matvec(pl[k], A[k], pr[k + 1], t)
    assert abs(np.vdot(v, f(u)) - np.vdot(u, f(v))) < 1e-13


def test_poincare_separation():
    """Orthonormal frame + SPD A -> local operator SPD with spectrum inside
    [lambda_min(A), lambda_max(A)] (PAPER.md:526 'Poincare Separation Theorem')."""
    d, n = 4, 2
    N = n * n
    rng = np.random.default_rng(51)
    Xf = ttgen.spd_factor(rng, d, n, 2)
    Zf = ttgen.spd_factor(rng, d, n, 2)
    A = ttgen.kron_sum_operator(Xf, Zf, n)
    Af = full_matrix(A)
    lam = np.linalg.eigvalsh((Af + Af.T) / 2)
    r = ttgen.capped_ranks(d, N, 6)
    x = ttgen.gaussian_tt_vector(rng, N, r)
    xl = ttgen.left_orthonormalise(x)
    xr = ttgen.right_orthonormalise(x)
    for k in range(d):
        mixed = xl[:k] + [x[k]] + xr[k + 1:]
        pl, _ = oracle.sweep_interfaces(mixed, A, 1)
        _, pr = oracle.sweep_interfaces(mixed, A, 2)
        shape = x[k].shape
        m = int(np.prod(shape))
        L = np.empty((m, m))
        for c in range(m):
            e = np.zeros(m)
            e[c] = 1.0
            L[:, c] = oracle.local_matvec(pl[k], A[k], pr[k + 1], e.reshape(shape)).reshape(-1)
        assert np.abs(L - L.T).max() < 1e-12
        mu = np.linalg.eigvalsh(L)
        assert mu.min() >= lam.min() - 1e-10 and mu.max() <= lam.max() + 1e-10


# --------------------------------------------------------------------------------------
# (B) batched
# --------------------------------------------------------------------------------------
def test_batched_columns_match_projected_operator():
    x, A, X = _rand_tt(61, 4, 4, [1, 4, 6, 4, 1], [1, 3, 5, 2, 1], nvec=5)
    Af = full_matrix(A)
    pl, pr = oracle.sweep_interfaces(x, A)
    for k in range(4):
        Y = oracle.local_matvec_batched(pl[k], A[k], pr[k + 1], X[k])
        P = projected_operator(x, Af, k)
        for m in range(5):
            ref = P @ X[k][:, :, m, :].reshape(-1)
            assert rel_fro(Y[:, :, m, :].reshape(-1), ref) < TOL_DENSE


# --------------------------------------------------------------------------------------
# (AP) operator apply
# --------------------------------------------------------------------------------------
@pytest.mark.parametrize("case", SMALL_CASES)
def test_operator_apply_brute_force(case):
    seed, d, N, r, R = case
    x, A, _ = _rand_tt(seed, d, N, r, R)
    z = oracle.operator_apply(x, A)
    for k in range(d):
        assert z[k].shape == (r[k] * R[k], N, r[k + 1] * R[k + 1])   # ranks multiply
    assert rel_fro(full_vector(z), full_matrix(A) @ full_vector(x)) < TOL_DENSE


def test_operator_apply_rectangular():
    """n_row != n_col is allowed by Def. TT Matrix."""
    rng = np.random.default_rng(71)
    x = ttgen.gaussian_tt_vector(rng, 3, [1, 2, 3, 1])
    A = [rng.standard_normal(s) for s in [(1, 5, 3, 2), (2, 2, 3, 4), (4, 4, 3, 1)]]
    z = oracle.operator_apply(x, A)
    assert rel_fro(full_vector(z), full_matrix(A) @ full_vector(x)) < TOL_DENSE


def test_diag_tt_hadamard():
    """apply(diag_TT(w), v) = w (.) v  (Def. TT Diagonalisation + Remark)."""
    rng = np.random.default_rng(81)
    w = ttgen.gaussian_tt_vector(rng, 4, [1, 3, 2, 2, 1])
    v = ttgen.gaussian_tt_vector(rng, 4, [1, 2, 4, 3, 1])
    D = []
    for c in w:
        r0, n, r1 = c.shape
        m = np.zeros((r0, n, n, r1))
        for i in range(n):
            m[:, i, i, :] = c[:, i, :]
        D.append(m)
    z = oracle.operator_apply(v, D)
    assert rel_fro(full_vector(z), full_vector(w) * full_vector(v)) < TOL_DENSE


@pytest.mark.parametrize("idx", [2])
def test_sylvester_apply_full_scale(idx):
    """Config 2 at full scale: (X (x) I + I (x) Z) vec_TT(M) = vec_TT(XM + MZ^T)
    (PAPER.md:313-331 vec_TT, 380-386 Kronecker, 449 L_X form)."""
    inp = ttgen.make_inputs(idx)
    d = inp.cfg.d
    n = 2
    Xd = full_matrix(inp.factors["X"])
    Zd = full_matrix(inp.factors["Z"])
    M = unvec_tt_dense(full_vector(inp.x), d, n)
    z = oracle.operator_apply(inp.x, inp.A)
    ref = vec_tt_dense(Xd @ M + M @ Zd.T, d, n)
    assert rel_fro(full_vector(z), ref) < TOL_DENSE


@pytest.mark.parametrize("idx", [2, 4])
def test_energy_full_scale_sylvester(idx):
    """Configs 2/4: phiL[d] = phiR[0] = <x, A x> = <M, XM + MZ> computed densely from the
    2^d x 2^d Sylvester form, and <x_k, y_k> equals it at every core."""
    inp = ttgen.make_inputs(idx)
    d = inp.cfg.d
    n = 2
    Xd = full_matrix(inp.factors["X"])
    Zd = full_matrix(inp.factors["Z"])
    M = unvec_tt_dense(full_vector(inp.x), d, n)
    e = float(np.sum(M * (Xd @ M + M @ Zd.T)))
    pl, pr = oracle.sweep_interfaces(inp.x, inp.A)
    assert abs(pl[d].item() - e) <= 1e-11 * abs(e)
    assert abs(pr[0].item() - e) <= 1e-11 * abs(e)
    for k in [0, d // 2, d - 1]:
        y = oracle.local_matvec(pl[k], inp.A[k], pr[k + 1], inp.x[k])
        assert abs(np.vdot(inp.x[k], y) - e) <= 1e-11 * abs(e)


# --------------------------------------------------------------------------------------
# golden closed forms (PAPER.md:609-631 MaxCut rank-1 operators)
# --------------------------------------------------------------------------------------
def _vec_tt_I(d, n):
    return [np.eye(n).reshape(1, n * n, 1).copy() for _ in range(d)]


def _vec_tt_J(d, n):
    return [np.ones((1, n * n, 1)) for _ in range(d)]


def _diag_tt(v):
    out = []
    for c in v:
        r0, N, r1 = c.shape
        m = np.zeros((r0, N, N, r1))
        for i in range(N):
            m[:, i, i, :] = c[:, i, :]
        out.append(m)
    return out


def _tt_vec_sum(a, b):
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


def test_golden_maxcut_rank1():
    g = json.load(open(os.path.join(GOLDEN, "maxcut_rank1_d3.json")))
    d, n = g["d"], g["n"]
    x = _vec_tt_J(d, n)
    Aeq = _diag_tt(_vec_tt_I(d, n))
    pl, pr = oracle.sweep_interfaces(x, Aeq)
    assert [p.item() for p in pl] == g["A_eq"]["phiL_scalar"]
    assert [p.item() for p in pr] == g["A_eq"]["phiR_scalar"]
    for k in range(d):
        y = oracle.local_matvec(pl[k], Aeq[k], pr[k + 1], x[k])
        assert y.reshape(-1).tolist() == g["A_eq"]["y_k"][k]
    assert pl[d].item() == g["A_eq"]["energy"]
    negI = _vec_tt_I(d, n)
    negI[0] = -negI[0]
    KY = _diag_tt(_tt_vec_sum(_vec_tt_J(d, n), negI))
    assert KY[1].shape[0] == 2                       # rank_TT(K_Y) = 2
    pl, pr = oracle.sweep_interfaces(x, KY)
    assert pl[d].item() == g["K_Y"]["energy"] == pr[0].item()
    for k in range(d):
        y = oracle.local_matvec(pl[k], KY[k], pr[k + 1], x[k])
        assert y.reshape(-1).tolist() == g["K_Y"]["y_k"][k]


# --------------------------------------------------------------------------------------
# error behaviour
# --------------------------------------------------------------------------------------
def test_oracle_rejects_bad_arguments():
    L = oracle.lib()
    assert L.tt_oracle_local_matvec(0, 4, 1, 1, 1, None, None, None, None, None) == 2
    buf = np.zeros(16)
    p = buf.ctypes.data
    assert L.tt_oracle_local_matvec(0, 4, 1, 1, 1, p, p, p, p, p) == 1
    assert L.tt_oracle_local_matvec(1, 4, 1, -1, 1, p, p, p, p, p) == 1
    assert L.tt_oracle_local_matvec(1 << 40, 1 << 20, 1 << 20, 1, 1, p, p, p, p, p) == 5


# --------------------------------------------------------------------------------------
# two-site (DMRG supercore) local matvec — SURVEY.md 8(f) row 4
# --------------------------------------------------------------------------------------
def _two_site_frame(x, k):
    """X_{!=k,k+1} = T^{<k} (x) I_{n_k} (x) I_{n_{k+1}} (x) T^{>k+1} (Def. Frame, two sites)."""
    from dense_ref import left_interface, right_interface
    n1, n2 = x[k].shape[1], x[k + 1].shape[1]
    return np.kron(np.kron(left_interface(x, k), np.eye(n1 * n2)), right_interface(x, k + 1))


@pytest.mark.parametrize("case", [(91, 4, 3, [1, 3, 4, 5, 1], [1, 2, 3, 2, 1]),
                                  (92, 5, 2, [1, 2, 4, 4, 2, 1], [1, 3, 2, 3, 2, 1])])
def test_two_site_matvec_projected_operator(case):
    seed, d, N, r, R = case
    x, A, _ = _rand_tt(seed, d, N, r, R)
    Af = full_matrix(A)
    pl, pr = oracle.sweep_interfaces(x, A)
    rng = np.random.default_rng(seed)
    for k in range(d - 1):
        w = rng.standard_normal((r[k], N, N, r[k + 2]))
        y = oracle.local_matvec_two_site(pl[k], A[k], A[k + 1], pr[k + 2], w)
        F = _two_site_frame(x, k)
        ref = F.T @ Af @ F @ w.reshape(-1)
        assert rel_fro(y.reshape(-1), ref) < TOL_DENSE, k


def test_two_site_merged_supercore_energy():
    """With w = the merged supercore x_k x_{k+1}, <w, y> = x^T A x (restricted energy)."""
    x, A, _ = _rand_tt(93, 4, 4, [1, 4, 6, 4, 1], [1, 3, 3, 3, 1])
    v = full_vector(x)
    e = v @ full_matrix(A) @ v
    pl, pr = oracle.sweep_interfaces(x, A)
    for k in range(3):
        w = np.einsum("aib,bjc->aijc", x[k], x[k + 1])
        y = oracle.local_matvec_two_site(pl[k], A[k], A[k + 1], pr[k + 2], w)
        assert abs(np.vdot(w, y) - e) <= 1e-12 * abs(e)


# --------------------------------------------------------------------------------------
# projected KKT block system
# --------------------------------------------------------------------------------------
KKT_TERMS = [  # (row, col, op, op2, coeff): the 3x3 system of PAPER.md:460-472
    (0, 0, 0, -1, -1.0),   # -W^T A_eq W
    (0, 1, 1, -1, 1.0),    #  W^T K_Y W
    (1, 0, 2, -1, -1.0),   # -W^T T A_ineq W
    (1, 2, 3, -1, 1.0),    #  W^T (R_ineq + K_T) W
    (2, 0, 4, -1, 1.0),    #  W^T L_Z W
    (2, 1, 5, 6, 1.0),     # (W^T L_X W)(W^T A_eq^T W)
    (2, 2, 5, 7, 1.0),     # (W^T L_X W)(W^T A_ineq^T W)
]


def test_block_local_matvec_dense():
    """The block action equals the dense 3x3 block matrix of projected operators (each
    X_{!=k}^T A_o X_{!=k} with the shared frame) times the block vector."""
    rng = np.random.default_rng(101)
    d, N = 4, 4
    r = [1, 4, 6, 4, 1]
    x = ttgen.gaussian_tt_vector(rng, N, r)
    Rs = [[1, 2, 3, 2, 1], [1, 1, 2, 1, 1], [1, 3, 2, 3, 1], [1, 2, 2, 2, 1],
          [1, 2, 3, 2, 1], [1, 3, 3, 3, 1], [1, 2, 1, 2, 1], [1, 1, 3, 1, 1]]
    Aops = [ttgen.gaussian_tt_matrix(rng, N, N, R) for R in Rs]
    k = 2
    ops = []
    dense = []
    for A in Aops:
        pl, pr = oracle.sweep_interfaces(x, A)
        ops.append((pl[k], A[k], pr[k + 1]))
        dense.append(projected_operator(x, full_matrix(A), k))
    nb = 3
    X = rng.standard_normal((r[k], N, nb, r[k + 1]))
    Y = oracle.block_local_matvec(ops, KKT_TERMS, X)
    m = r[k] * N * r[k + 1]
    big = np.zeros((nb * m, nb * m))
    for (row, col, op, op2, c) in KKT_TERMS:
        blk = dense[op] @ (dense[op2] if op2 >= 0 else np.eye(m))
        big[row * m:(row + 1) * m, col * m:(col + 1) * m] += c * blk
    xv = np.concatenate([X[:, :, b, :].ravel() for b in range(nb)])
    yv = big @ xv
    for b in range(nb):
        assert rel_fro(Y[:, :, b, :].ravel(), yv[b * m:(b + 1) * m]) < TOL_DENSE
