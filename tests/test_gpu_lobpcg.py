"""GPU parity for the matrix-free block LOBPCG of the step-length local eigenproblem
 against oracle/geneig.py.

The eigenvalues of the projected pencil are unique: they are compared with the oracle's
Cholesky-reduced dense eigensolve.  Eigenvectors are compared through what is unique or
checkable: the residual ||L_A x - lam L_B x|| computed by the ORACLE's operators and
L_B-orthonormality.
"""
import numpy as np
import pytest

import oracle
import ttgen
from oracle.geneig import (block_columns, columns_block, geneig_dense, local_geneig,
                           local_operator_dense, step_length)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


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


def mixed_frame(x, k, two_site=False):
    xl, xr = ttgen.left_orthonormalise(x), ttgen.right_orthonormalise(x)
    last = k + 1 if two_site else k
    return xl[:k] + [x[j] for j in range(k, last + 1)] + xr[last + 1:]


def neg(cores):
    out = [c.copy() for c in cores]
    out[0] = -out[0]
    return out


def step_system(seed, d=8, rE=8, rM=3, rdM=3, fro=6.0, k=3, two_site=False):
    """E train (mode 2) in mixed-canonical form, M = X (SPD), dM = dX (symmetric): the pencil
    (-dX, X) of the primal step length (reading R12)."""
    rng = np.random.default_rng(seed)
    n = 2
    x = ttgen.gaussian_tt_vector(rng, n, ttgen.capped_ranks(d, n, rE))
    M = ttgen.spd_factor(rng, d, n, rM)
    dM = ttgen.symmetric_tt_matrix(rng, d, n, rdM, fro=fro)
    mixed = mixed_frame(x, k, two_site)
    return rng, mixed, neg(dM), M


def local_triplets(mixed, op, k, two_site=False):
    pl, pr = oracle.sweep_interfaces(mixed, op, 3)
    return pl[k], pr[k + 2 if two_site else k + 1]


def check_pairs(LA, LB, V, lam, tol):
    """Residual and L_B-orthonormality of the GPU Ritz pairs, with the oracle's matrices."""
    B = np.eye(LA.shape[0]) if LB is None else LB
    R = LA @ V - (B @ V) * lam
    scale = np.abs(LA).max() + np.abs(lam).max() * np.abs(B).max()
    assert np.abs(R).max() <= tol * scale * np.sqrt(LA.shape[0])
    assert np.allclose(V.T @ B @ V, np.eye(V.shape[1]), atol=1e-9)


@pytest.mark.parametrize("nb", [1, 4])
def test_lobpcg_standard_vs_oracle(tt, nb):
    rng, mixed, A, _ = step_system(51)
    k = 3
    phiL, phiR = local_triplets(mixed, A, k)
    op = (phiL, A[k], phiR)
    rl, n, rr = phiL.shape[0], A[k].shape[1], phiR.shape[0]
    X0 = rng.standard_normal((rl, n, nb, rr))
    X, lam, res, its, step = tt.tt_local_lobpcg(tuple(g(t) for t in op), g(X0), maxiter=600,
                                                tol=1e-11)
    torch.cuda.synchronize()
    ref, _ = local_geneig(op, None, nb)
    LA = local_operator_dense(*op)
    assert np.allclose(h(lam), ref, rtol=0, atol=1e-10 * np.abs(ref).max())
    assert h(res).max() <= 1e-11 and 0 < int(h(its)[0]) < 600
    check_pairs(LA, None, block_columns(h(X)), h(lam), 1e-10)


@pytest.mark.parametrize("nb", [1, 3])
def test_lobpcg_step_length_generalised(tt, nb):
    rng, mixed, negdX, M = step_system(52, fro=20.0)
    k = 4
    pA = local_triplets(mixed, negdX, k)
    pB = local_triplets(mixed, M, k)
    opA, opB = (pA[0], negdX[k], pA[1]), (pB[0], M[k], pB[1])
    rl, n, rr = pA[0].shape[0], 2, pA[1].shape[0]
    X0 = rng.standard_normal((rl, n, nb, rr))
    X, lam, res, its, step = tt.tt_local_lobpcg(tuple(g(t) for t in opA), g(X0),
                                                opB=tuple(g(t) for t in opB), maxiter=800,
                                                tol=1e-11)
    torch.cuda.synchronize()
    ref, _ = local_geneig(opA, opB, nb)
    assert np.allclose(h(lam), ref, rtol=0, atol=1e-10 * np.abs(ref).max())
    assert abs(float(h(step)[0]) - step_length(ref[0])) <= 1e-10
    assert h(res).max() <= 1e-11
    check_pairs(local_operator_dense(*opA), local_operator_dense(*opB), block_columns(h(X)),
                h(lam), 1e-10)


def test_merge_operator_cores(tt):
    rng = np.random.default_rng(53)
    A1 = rng.standard_normal((3, 2, 2, 5))
    A2 = rng.standard_normal((5, 2, 2, 4))
    got = h(tt.tt_merge_operator_cores(g(A1), g(A2)))
    ref = np.einsum("aijg,gklb->aikjlb", A1, A2).reshape(3, 4, 4, 4)
    assert np.abs(got - ref).max() <= 1e-14 * np.abs(ref).max()


def _dense_two_site(phiL, A1, A2, phiR):
    """Dense two-site local operator from the ORACLE's two-site matvec on unit vectors."""
    rl, n1, n2, rr = phiL.shape[0], A1.shape[1], A2.shape[1], phiR.shape[0]
    m = rl * n1 * n2 * rr
    cols = []
    for e in range(m):
        u = np.zeros(m)
        u[e] = 1.0
        cols.append(oracle.local_matvec_two_site(phiL, A1, A2, phiR,
                                                 u.reshape(rl, n1, n2, rr)).ravel())
    return np.array(cols).T


def test_lobpcg_two_site_vs_oracle(tt):
    """DMRG-style two-site step-length eigenproblem: supercore operators merged
    on the GPU, dense reference from the oracle's two-site matvec."""
    rng, mixed, negdX, M = step_system(54, d=7, rE=6, k=2, two_site=True, fro=15.0)
    k = 2
    pA = local_triplets(mixed, negdX, k, True)
    pB = local_triplets(mixed, M, k, True)
    LA = _dense_two_site(pA[0], negdX[k], negdX[k + 1], pA[1])
    LB = _dense_two_site(pB[0], M[k], M[k + 1], pB[1])
    A12 = tt.tt_merge_operator_cores(g(negdX[k]), g(negdX[k + 1]))
    M12 = tt.tt_merge_operator_cores(g(M[k]), g(M[k + 1]))
    rl, rr = pA[0].shape[0], pA[1].shape[0]
    nb = 2
    X0 = rng.standard_normal((rl, 4, nb, rr))
    X, lam, res, its, step = tt.tt_local_lobpcg((g(pA[0]), A12, g(pA[1])), g(X0),
                                                opB=(g(pB[0]), M12, g(pB[1])), maxiter=800,
                                                tol=1e-11)
    torch.cuda.synchronize()
    ref, _ = geneig_dense(LA, LB, nb)
    assert np.allclose(h(lam), ref, rtol=0, atol=1e-10 * np.abs(ref).max())
    assert abs(float(h(step)[0]) - step_length(ref[0])) <= 1e-10
    check_pairs(LA, LB, block_columns(h(X)), h(lam), 1e-10)


def test_lobpcg_kron_sum_closed_form(tt):
    """Full orthonormal frame: GPU Ritz values equal the closed-form Kronecker-sum spectrum."""
    rng = np.random.default_rng(55)
    d, n = 4, 2
    f = np.array([-0.4, 1.3])
    Q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    F = Q @ np.diag(f) @ Q.T
    I = np.eye(n)
    A = [np.stack([F, I], -1)[None]]
    mid = np.zeros((2, n, n, 2))
    mid[0, :, :, 0], mid[1, :, :, 0], mid[1, :, :, 1] = I, F, I
    A += [mid, mid.copy()]
    last = np.zeros((2, n, n, 1))
    last[0, :, :, 0], last[1, :, :, 0] = I, F
    A.append(last)
    x = ttgen.gaussian_tt_vector(rng, n, [1, 2, 4, 2, 1])
    k = 2
    mixed = mixed_frame(x, k)
    phiL, phiR = local_triplets(mixed, A, k)
    sums = np.sort([f[list(i)].sum() for i in np.ndindex(*([2] * d))])[::-1]
    X0 = rng.standard_normal((4, 2, 3, 2))
    X, lam, res, its, step = tt.tt_local_lobpcg((g(phiL), g(A[k]), g(phiR)), g(X0), maxiter=200,
                                                tol=1e-12)
    torch.cuda.synchronize()
    # the top eigenvalue 4 * 1.3 is simple; the next (3 * 1.3 - 0.4) has multiplicity 4
    assert np.allclose(h(lam), sums[:3], rtol=0, atol=1e-12)


def test_lobpcg_maxiter0_is_rayleigh_ritz(tt):
    """maxiter = 0: the Ritz pairs of the initial block (oracle: dense pencil projected on the
    block, solved by the Cholesky-reduced eigensolve)."""
    rng, mixed, A, _ = step_system(56)
    k = 3
    phiL, phiR = local_triplets(mixed, A, k)
    op = (phiL, A[k], phiR)
    rl, rr = phiL.shape[0], phiR.shape[0]
    nb = 4
    X0 = rng.standard_normal((rl, 2, nb, rr))
    X, lam, res, its, step = tt.tt_local_lobpcg(tuple(g(t) for t in op), g(X0.copy()), maxiter=0)
    torch.cuda.synchronize()
    V0 = block_columns(X0)
    LA = local_operator_dense(*op)
    ref, _ = geneig_dense(V0.T @ LA @ V0, V0.T @ V0, nb)
    assert np.allclose(h(lam), ref, rtol=0, atol=1e-11 * np.abs(ref).max())
    assert int(h(its)[0]) == 0


def test_lobpcg_early_stop_and_graph_capture(tt):
    """Convergence gates the remaining iterations (iters < maxiter); a CUDA-graph replay of the
    call reproduces the eager result bit for bit (fixed launch sequence, deterministic)."""
    rng, mixed, A, _ = step_system(57)
    k = 3
    phiL, phiR = local_triplets(mixed, A, k)
    op = tuple(g(t) for t in (phiL, A[k], phiR))
    rl, rr = phiL.shape[0], phiR.shape[0]
    X0 = g(rng.standard_normal((rl, 2, 2, rr)))
    ws = torch.empty(tt.tt_local_lobpcg_workspace_size(rl, 2, rr, A[k].shape[0], A[k].shape[3],
                                                       0, 0, 2), dtype=torch.uint8, device="cuda")
    Xe = X0.clone()
    _, lam_e, res_e, its_e, _ = tt.tt_local_lobpcg(op, Xe, maxiter=3000, tol=1e-9, workspace=ws)
    torch.cuda.synchronize()
    assert int(h(its_e)[0]) < 3000 and h(res_e).max() <= 1e-9
    Xg = X0.clone()
    lam_g = torch.empty(2, dtype=torch.float64, device="cuda")
    res_g = torch.empty_like(lam_g)
    its_g = torch.empty(1, dtype=torch.int64, device="cuda")
    st_g = torch.empty(1, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            tt.tt_local_lobpcg(op, Xg, maxiter=3000, tol=1e-9, lam=lam_g, res=res_g, iters=its_g,
                               step=st_g, workspace=ws, stream=s)
    Xg.copy_(X0)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(Xg, Xe) and torch.equal(lam_g, lam_e) and torch.equal(its_g, its_e)


def test_lobpcg_errors(tt):
    rng, mixed, A, M = step_system(58)
    k = 3
    phiL, phiR = local_triplets(mixed, A, k)
    op = tuple(g(t) for t in (phiL, A[k], phiR))
    rl, rr = phiL.shape[0], phiR.shape[0]
    with pytest.raises(tt.TTError):
        tt.tt_local_lobpcg(op, g(np.zeros((rl, 2, 33, rr))))
    lib = tt.lib
    X = g(rng.standard_normal((rl, 2, 2, rr)))
    lam = torch.empty(2, dtype=torch.float64, device="cuda")
    res = torch.empty_like(lam)
    its = torch.empty(1, dtype=torch.int64, device="cuda")
    RlA, RrA = A[k].shape[0], A[k].shape[3]
    need = tt.tt_local_lobpcg_workspace_size(rl, 2, rr, RlA, RrA, 0, 0, 2)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    args = lambda pB, wsb: (rl, 2, rr, RlA, RrA, RlA, RrA, 2, 10, 20, 1e-9, op[0].data_ptr(),
                            op[1].data_ptr(), op[2].data_ptr(), *pB, X.data_ptr(),
                            lam.data_ptr(), res.data_ptr(), its.data_ptr(), None,
                            ws.data_ptr(), wsb, None)
    assert lib.tt_local_lobpcg(*args((op[0].data_ptr(), None, None), need)) == 2   # NULL_POINTER
    assert lib.tt_local_lobpcg(*args((None, None, None), need - 1)) == 4            # WORKSPACE
    assert lib.tt_local_lobpcg(*args((None, None, None), need)) == 0
    torch.cuda.synchronize()


def test_lobpcg_max_block(tt):
    """nb = 32 (the largest block): Rayleigh-Ritz on s = 96 columns in one CTA."""
    rng, mixed, A, _ = step_system(59, d=8, rE=12)
    k = 4
    phiL, phiR = local_triplets(mixed, A, k)
    op = (phiL, A[k], phiR)
    rl, rr = phiL.shape[0], phiR.shape[0]
    nb = 32
    X0 = rng.standard_normal((rl, 2, nb, rr))
    X, lam, res, its, step = tt.tt_local_lobpcg(tuple(g(t) for t in op), g(X0), maxiter=400,
                                                tol=1e-10)
    torch.cuda.synchronize()
    ref, _ = local_geneig(op, None, nb)
    assert np.allclose(h(lam), ref, rtol=0, atol=1e-9 * np.abs(ref).max())
    check_pairs(local_operator_dense(*op), None, block_columns(h(X)), h(lam), 1e-9)
