"""GPU parity for the Petrov-Galerkin local operations (bra train != ket train) and the AMEn
enrichment against oracle/petrov.py."""
import numpy as np
import pytest

import ttgen
from dense_ref import full_vector, rel_fro
from oracle.petrov import enrich_right, interface_left_pg, interface_right_pg, local_matvec_pg

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-11


@pytest.fixture(scope="module")
def tt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2509_11890_b200 as m
    return m


def g(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def h(t):
    return t.detach().cpu().numpy()


# (rl_bra, rl, n, rr_bra, rr, Rl, Rr, nvec): ragged, bra wider and narrower than ket,
# interior-core scale
SHAPES = [(3, 5, 4, 2, 7, 3, 2, 1), (17, 9, 4, 33, 12, 5, 4, 3), (64, 48, 4, 32, 80, 16, 9, 2),
          (256, 128, 4, 64, 256, 36, 36, 4), (8, 64, 16, 8, 64, 4, 4, 1)]


@pytest.mark.parametrize("shape", SHAPES)
def test_pg_matvec_vs_oracle(tt, shape):
    rlb, rl, n, rrb, rr, Rl, Rr, K = shape
    rng = np.random.default_rng(71)
    phiL, A = rng.standard_normal((rlb, Rl, rl)), rng.standard_normal((Rl, n, n, Rr))
    phiR, X = rng.standard_normal((rrb, Rr, rr)), rng.standard_normal((rl, n, K, rr))
    Y = h(tt.tt_local_matvec_pg(g(phiL), g(A), g(phiR), g(X)))
    assert rel_fro(Y, local_matvec_pg(phiL, A, phiR, X)) <= TOL


@pytest.mark.parametrize("shape", SHAPES)
def test_pg_interfaces_vs_oracle(tt, shape):
    rlb, rl, n, rrb, rr, Rl, Rr, _ = shape
    rng = np.random.default_rng(72)
    A = rng.standard_normal((Rl, n, n, Rr))
    xb, xk = rng.standard_normal((rlb, n, rrb)), rng.standard_normal((rl, n, rr))
    phiL, phiR = rng.standard_normal((rlb, Rl, rl)), rng.standard_normal((rrb, Rr, rr))
    L = h(tt.tt_interface_left_pg(g(phiL), g(A), g(xb), g(xk)))
    assert rel_fro(L, interface_left_pg(phiL, A, xb, xk)) <= TOL
    R = h(tt.tt_interface_right_pg(g(phiR), g(A), g(xb), g(xk)))
    assert rel_fro(R, interface_right_pg(phiR, A, xb, xk)) <= TOL


def test_pg_square_equals_galerkin_path(tt):
    """bra == ket: the Petrov-Galerkin calls agree with the Galerkin hot path (both GPU)."""
    rng = np.random.default_rng(73)
    a, n, b, Rl, Rr, K = 64, 4, 48, 9, 16, 3
    phiL, A = g(rng.standard_normal((a, Rl, a))), g(rng.standard_normal((Rl, n, n, Rr)))
    phiR, X = g(rng.standard_normal((b, Rr, b))), g(rng.standard_normal((a, n, K, b)))
    Y1 = tt.tt_local_matvec_pg(phiL, A, phiR, X)
    Y2 = torch.empty_like(X)
    tt.tt_local_matvec_batched(phiL, A, phiR, X, Y2)
    assert rel_fro(h(Y1), h(Y2)) <= 1e-13
    x = g(rng.standard_normal((a, n, b)))
    assert rel_fro(h(tt.tt_interface_left_pg(phiL, A, x, x)), h(tt.tt_interface_left(phiL, A, x))) <= 1e-13


def test_enrich_right_vs_oracle(tt):
    rng = np.random.default_rng(74)
    x = ttgen.gaussian_tt_vector(rng, 4, [1, 4, 16, 24, 16, 4, 1])
    k = 2
    zk = rng.standard_normal((16, 4, 5))
    xk, x1 = (h(t) for t in tt.tt_enrich_right(g(x[k]), g(zk), g(x[k + 1])))
    rk, r1 = enrich_right(x[k], zk, x[k + 1])
    assert xk.shape == rk.shape == (16, 4, 29) and x1.shape == r1.shape
    M = xk.reshape(64, -1)
    assert np.abs(M.T @ M - np.eye(29)).max() <= 1e-11
    y = x[:k] + [xk, x1] + x[k + 2:]
    assert rel_fro(full_vector(y), full_vector(x)) <= 1e-11
    P = M @ M.T
    for c in (x[k].reshape(64, -1), zk.reshape(64, -1)):
        assert np.abs(P @ c - c).max() <= 1e-10 * np.abs(c).max()


def test_enrich_right_async_equals_sync(tt):
    """Device-side rank into zero-padded outputs: the padded pair is the enriched train as it
    stands, the rank equals the synchronous call's; a rank-deficient residual (z_k inside the
    span of x_k) is truncated away on the device."""
    rng = np.random.default_rng(75)
    x = ttgen.gaussian_tt_vector(rng, 4, [1, 4, 16, 24, 16, 4, 1])
    k = 2
    for zk in (rng.standard_normal((16, 4, 5)),
               np.einsum("aib,bc->aic", x[k], rng.standard_normal((24, 3)))):
        xs, x1s = (h(t) for t in tt.tt_enrich_right(g(x[k]), g(zk), g(x[k + 1]), 1e-10))
        xa, x1a, rank = tt.tt_enrich_right_async(g(x[k]), g(zk), g(x[k + 1]), 1e-10)
        s = int(rank.item())
        xa, x1a = h(xa), h(x1a)
        assert s == xs.shape[2]
        assert xa.shape[2] == min(64, 24 + zk.shape[2]) == x1a.shape[0]
        assert not xa[:, :, s:].any() and not x1a[s:].any()
        y = x[:k] + [xa, x1a] + x[k + 2:]
        assert rel_fro(full_vector(y), full_vector(x)) <= 1e-11
        M = xa[:, :, :s].reshape(64, s)
        assert np.abs(M.T @ M - np.eye(s)).max() <= 1e-9


def test_amen_residual_enrichment_step(tt):
    """One AMEn enrichment step at core k of a left-to-right sweep: the residual
    core r_k = X^{<k},Z^{>k}-projection of (b - A x) -- the projected right-hand side minus the
    Petrov-Galerkin matvec -- computed on the GPU from two-train interfaces, then x_k enriched.
    Checked against the same pipeline in the oracle."""
    rng = np.random.default_rng(75)
    d, N = 5, 4
    x = ttgen.left_orthonormalise(ttgen.gaussian_tt_vector(rng, N, ttgen.capped_ranks(d, N, 6)))
    z = ttgen.gaussian_tt_vector(rng, N, ttgen.capped_ranks(d, N, 3))     # residual approx.
    bt = ttgen.gaussian_tt_vector(rng, N, ttgen.capped_ranks(d, N, 4))    # right-hand side
    A = ttgen.gaussian_tt_matrix(rng, N, N, ttgen.capped_ranks(d, N * N, 3))
    I = ttgen.identity_operator(d, N)
    k = 2
    # oracle: left interfaces bra x / ket x (A) and bra x / ket b (I); right bra z
    def chain_left(bra, ket, op):
        p = [np.ones((1, 1, 1))]
        for j in range(k):
            p.append(interface_left_pg(p[-1], op[j], bra[j], ket[j]))
        return p[k]

    def chain_right(bra, ket, op):
        p = np.ones((1, 1, 1))
        for j in range(d - 1, k, -1):
            p = interface_right_pg(p, op[j], bra[j], ket[j])
        return p
    rk_ref = (local_matvec_pg(chain_left(x, bt, I), I[k], chain_right(z, bt, I), bt[k]) -
              local_matvec_pg(chain_left(x, x, A), A[k], chain_right(z, x, A), x[k]))
    xk_ref, x1_ref = enrich_right(x[k], rk_ref, x[k + 1])
    # GPU
    G = lambda cores: [g(c) for c in cores]
    gx, gz, gb, gA, gI = G(x), G(z), G(bt), G(A), G(I)

    def gchain_left(bra, ket, op):
        p = g(np.ones((1, 1, 1)))
        for j in range(k):
            p = tt.tt_interface_left_pg(p, op[j], bra[j], ket[j])
        return p

    def gchain_right(bra, ket, op):
        p = g(np.ones((1, 1, 1)))
        for j in range(d - 1, k, -1):
            p = tt.tt_interface_right_pg(p, op[j], bra[j], ket[j])
        return p
    f = tt.tt_local_matvec_pg(gchain_left(gx, gb, gI), gI[k], gchain_right(gz, gb, gI), gb[k])
    ax = tt.tt_local_matvec_pg(gchain_left(gx, gx, gA), gA[k], gchain_right(gz, gx, gA), gx[k])
    rk = f - ax
    assert rel_fro(h(rk), rk_ref) <= 1e-10
    xk, x1 = (h(t) for t in tt.tt_enrich_right(gx[k], rk.contiguous(), gx[k + 1]))
    assert xk.shape == xk_ref.shape
    y = x[:k] + [xk, x1] + x[k + 2:]
    assert rel_fro(full_vector(y), full_vector(x)) <= 1e-11
    P, Pr = xk.reshape(-1, xk.shape[2]), xk_ref.reshape(-1, xk_ref.shape[2])
    assert np.abs(P @ P.T - Pr @ Pr.T).max() <= 1e-9
