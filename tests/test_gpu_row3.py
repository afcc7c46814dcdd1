"""GPU parity for SURVEY.md §8(f) row 3 beyond rounding: core orthonormalisation and the
block-index move against oracle/rounding.py.

SVD factors are unique only up to signs/rotations, so the comparisons are on what is unique:
the represented (block) tensors, the truncation rank, orthonormality, and orthogonal
projectors onto the kept singular subspaces (gapped spectra)."""
import numpy as np
import pytest

import ttgen
from dense_ref import full_vector, left_interface, rel_fro
from oracle.rounding import (block_move_left, block_move_right, orthonormalise_left,
                             orthonormalise_right)

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


def _graded(rng, m, q, sig):
    U = np.linalg.qr(rng.standard_normal((m, len(sig))))[0]
    V = np.linalg.qr(rng.standard_normal((q, len(sig))))[0]
    return (U * sig) @ V.T


@pytest.mark.parametrize("direction", ["left", "right"])
def test_orthonormalise_vs_oracle(tt, direction):
    rng = np.random.default_rng(31)
    d, N = 6, 4
    x = ttgen.gaussian_tt_vector(rng, N, ttgen.capped_ranks(d, N, 12))
    flag = tt.TT_SWEEP_LEFT if direction == "left" else tt.TT_SWEEP_RIGHT
    out = [h(c) for c in tt.tt_orthonormalise([g(c) for c in x], flag)]
    ref = orthonormalise_left(x) if direction == "left" else orthonormalise_right(x)
    assert [c.shape for c in out] == [c.shape for c in ref]
    assert rel_fro(full_vector(out), full_vector(x)) <= 1e-11
    ks = range(d - 1) if direction == "left" else range(1, d)
    for k in ks:
        c = out[k]
        M = c.reshape(-1, c.shape[2]) if direction == "left" else c.reshape(c.shape[0], -1).T
        # the factorisations go through Gram matrices: orthonormality to ~ eps kappa^2
        assert np.abs(M.T @ M - np.eye(M.shape[1])).max() <= 1e-11
    if direction == "left":   # the left interfaces span the same subspaces as the oracle's
        for k in (1, 2, 3):
            A, B = left_interface(out, k), left_interface(ref, k)
            assert np.abs(A @ A.T - B @ B.T).max() <= 1e-11


@pytest.mark.parametrize("shape", [(3, 4, 4, 5, 4, 2), (16, 4, 2, 40, 4, 8), (8, 4, 4, 4, 4, 16)])
def test_block_move_right_exact(tt, shape):
    r0, n0, l, r1, n1, r2 = shape
    rng = np.random.default_rng(32)
    Wk_hat = rng.standard_normal((r0, n0, l, r1))
    Wk1 = rng.standard_normal((r1, n1, r2))
    Wk, W1 = tt.tt_block_move_right(g(Wk_hat), g(Wk1))
    Wk, W1 = h(Wk), h(W1)
    rk, r1k = block_move_right(Wk_hat, Wk1)
    assert Wk.shape == rk.shape and W1.shape == r1k.shape
    M = Wk.reshape(r0 * n0, -1)
    assert np.abs(M.T @ M - np.eye(M.shape[1])).max() <= 1e-11
    T0 = np.einsum("ailb,bjc->ailjc", Wk_hat, Wk1)
    assert rel_fro(np.einsum("ais,sjlc->ailjc", Wk, W1), T0) <= 1e-11


@pytest.mark.parametrize("delta", [1e-2, 1e-4])
@pytest.mark.parametrize("m_lt_q", [True, False])
def test_block_move_right_truncated(tt, delta, m_lt_q):
    rng = np.random.default_rng(33)
    r0, n0, l, r1, n1, r2 = (4, 4, 4, 8, 4, 3) if m_lt_q else (16, 4, 2, 6, 4, 3)
    sig = np.array([3.0, 2.0, 1.0, 0.5, 1e-3, 5e-4, 1e-6, 1e-7])
    Wk_hat = _graded(rng, r0 * n0, l * r1, sig).reshape(r0, n0, l, r1)
    Wk1 = rng.standard_normal((r1, n1, r2))
    Wk, W1 = (h(t) for t in tt.tt_block_move_right(g(Wk_hat), g(Wk1), delta))
    rk, r1k = block_move_right(Wk_hat, Wk1, delta)
    assert Wk.shape == rk.shape
    P, Pr = Wk.reshape(r0 * n0, -1), rk.reshape(r0 * n0, -1)
    # the kept singular subspace through the Gram matrix: accurate to ~ eps kappa^2,
    # kappa = sigma_max / sigma_min(kept)
    kappa = sig[0] / sig[Wk.shape[2] - 1]
    assert np.abs(P @ P.T - Pr @ Pr.T).max() <= 1e-13 * kappa ** 2
    T = np.einsum("ais,sjlc->ailjc", Wk, W1)
    Tr = np.einsum("ais,sjlc->ailjc", rk, r1k)
    assert rel_fro(T, Tr) <= 1e-10


@pytest.mark.parametrize("shape", [(2, 4, 5, 4, 3, 6), (8, 4, 32, 4, 4, 8)])
def test_block_move_left_vs_oracle(tt, shape):
    r0, n0, r1, n1, l, r2 = shape
    rng = np.random.default_rng(34)
    Wkm1 = rng.standard_normal((r0, n0, r1))
    Wk_hat = rng.standard_normal((r1, n1, l, r2))
    Wh, Wk = (h(t) for t in tt.tt_block_move_left(g(Wkm1), g(Wk_hat)))
    rh, rk = block_move_left(Wkm1, Wk_hat)
    assert Wh.shape == rh.shape and Wk.shape == rk.shape
    R = Wk.reshape(Wk.shape[0], -1)
    assert np.abs(R @ R.T - np.eye(R.shape[0])).max() <= 1e-11
    T0 = np.einsum("ajb,bilc->ajilc", Wkm1, Wk_hat)
    assert rel_fro(np.einsum("ajls,sic->ajilc", Wh, Wk), T0) <= 1e-11


def test_block_move_config5_size(tt):
    """Interior core of config 5 with the 4-component KKT block index:
    (256, 4, 4, 256) -> 1024 x 1024 unfolding, delta = 1e-6 on a graded spectrum."""
    rng = np.random.default_rng(35)
    r0 = r1 = 256
    sig = np.concatenate([np.geomspace(1.0, 1e-3, 200), np.geomspace(1e-9, 1e-12, 56)])
    Wk_hat = _graded(rng, r0 * 4, 4 * r1, sig).reshape(r0, 4, 4, r1)
    Q = np.linalg.qr(rng.standard_normal((4 * 1024, r1)))[0]    # (n1 r2) x r1, orthonormal
    Wk1 = np.ascontiguousarray(Q.T.reshape(r1, 4, 1024))
    Wk, W1 = (h(t) for t in tt.tt_block_move_right(g(Wk_hat), g(np.ascontiguousarray(Wk1)),
                                                   1e-6))
    rk, r1k = block_move_right(Wk_hat, Wk1, 1e-6)
    assert Wk.shape[2] == rk.shape[2] == 200
    P, Pr = Wk.reshape(1024, -1), rk.reshape(1024, -1)
    kappa = 1e3
    assert np.abs(P.T @ P - np.eye(200)).max() <= 1e-13 * kappa ** 2
    assert np.abs(P @ P.T - Pr @ Pr.T).max() <= 1e-13 * kappa ** 2
    T = np.einsum("ais,sjlc->ailjc", Wk, W1)
    Tr = np.einsum("ais,sjlc->ailjc", rk, r1k)
    assert rel_fro(T, Tr) <= 1e-10


def test_block_move_errors(tt):
    import ctypes
    buf = torch.zeros(16, dtype=torch.float64, device="cuda")
    p = buf.data_ptr()
    s_out = ctypes.c_int64()
    # both sides of the unfolding above 2048: refused before the workspace is examined
    assert tt.lib.tt_block_move_right(64, 64, 64, 64, 2, 2, 0.0, 0, p, p + 8, p + 16, p + 24,
                                      ctypes.byref(s_out), None, 0, None) == 1
    # NULL workspace
    assert tt.lib.tt_block_move_right(3, 4, 2, 5, 4, 2, 0.0, 0, p, p + 8, p + 16, p + 24,
                                      ctypes.byref(s_out), None, 0, None) == 4
    # aliasing output/input
    assert tt.lib.tt_block_move_left(3, 4, 5, 4, 2, 2, 0.0, 0, p, p + 8, p, p + 24,
                                     ctypes.byref(s_out), None, 0, None) == 3


@pytest.mark.parametrize("direction", ["left", "right"])
def test_orthonormalise_exact_on_graded_cores(tt, direction):
    """Householder QR (tt_qr.cuh): orthonormal to working precision and the represented tensor
    unchanged even when every unfolding has singular values from 1 down to 1e-14 (the Gram
    route squares that condition number: directions below ~1e-8 are lost)."""
    rng = np.random.default_rng(77)
    d, N = 6, 4
    ranks = ttgen.capped_ranks(d, N, 16)
    x = ttgen.gaussian_tt_vector(rng, N, ranks)
    for k in range(d):   # grade both bonds of every core
        x[k] = x[k] * np.logspace(0, -14, x[k].shape[2])[None, None, :]
        x[k] = x[k] * np.logspace(0, -7, x[k].shape[0])[:, None, None]
    flag = tt.TT_SWEEP_LEFT if direction == "left" else tt.TT_SWEEP_RIGHT
    out = [h(c) for c in tt.tt_orthonormalise([g(c) for c in x], flag)]
    v, vg = full_vector(x), full_vector(out)
    assert rel_fro(vg, v) <= 1e-12
    ks = range(d - 1) if direction == "left" else range(1, d)
    for k in ks:
        c = out[k]
        M = c.reshape(-1, c.shape[2]) if direction == "left" else c.reshape(c.shape[0], -1).T
        assert np.abs(M.T @ M - np.eye(M.shape[1])).max() <= 1e-13


@pytest.mark.parametrize("shape", [(1024, 256), (256, 256), (64, 256), (1000, 37), (5, 3), (33, 64)])
def test_cluster_qr_vs_gram_route(tt, shape):
    """The QR path against the Gram route (debug bit 29) on one two-core train whose first
    unfolding has the given shape: same represented tensor, both orthonormal."""
    m, c = shape
    rng = np.random.default_rng(m + c)
    n0 = 4
    r0 = max(1, m // n0)
    x = [rng.standard_normal((1, n0, r0)), rng.standard_normal((r0, n0, c)) / np.sqrt(r0 * n0),
         rng.standard_normal((c, n0, 1))]
    x[0] = x[0] / np.linalg.norm(x[0])
    outs = []
    for flags in (0, 1 << 29):
        tt.tt_debug_set_flags(flags)
        try:
            outs.append([h(t) for t in tt.tt_orthonormalise([g(t) for t in x], tt.TT_SWEEP_LEFT)])
        finally:
            tt.tt_debug_set_flags(0)
    for out in outs:
        assert rel_fro(full_vector(out), full_vector(x)) <= 1e-11
        M = out[1].reshape(-1, out[1].shape[2])
        assert np.abs(M.T @ M - np.eye(M.shape[1])).max() <= 1e-12
    assert rel_fro(full_vector(outs[0]), full_vector(outs[1])) <= 1e-11


@pytest.mark.parametrize("rows,c,kappa,pre", [
    (256, 256, 1e2, False), (256, 256, 1e2, True), (256, 256, 1e14, True), (64, 200, 1e10, True),
    (37, 37, 1e15, True), (256, 100, 1e12, True), (256, 100, 1e6, False), (5, 3, 1e3, False)])
def test_cluster_jacobi_svd_relative_accuracy(tt, rows, c, kappa, pre):
    """One-sided Jacobi (tt_qr.cuh): B J has orthogonal columns, J is orthogonal, B = BJ J^T, and
    the singular values are relatively accurate even at condition 1e14-1e15 (the Gram route
    resolves nothing below ~1e-8 of the largest).  B = U diag(s) V^T with known s; with `pre`,
    B is replaced by R^T of B's QR (same singular values) as tt_round's accurate route does:
    there Jacobi converges in a few sweeps at any condition (on B itself the count grows with
    the condition, 11 -> 26 sweeps from 1e2 to 1e14 for n = 64 in a numpy model of the order)."""
    rng = np.random.default_rng(rows * 7 + c)
    k = min(rows, c)
    s = np.logspace(0, -np.log10(kappa), k)
    U = np.linalg.qr(rng.standard_normal((rows, k)))[0]
    V = np.linalg.qr(rng.standard_normal((c, k)))[0]
    B = (U * s) @ V.T
    if pre:
        B = np.ascontiguousarray(np.linalg.qr(B)[1].T)
        rows, c = B.shape
    BJ, J, sig, sw = tt.tt_debug_svd(g(B))
    BJ, J, sig = h(BJ), h(J), h(sig)
    assert int(h(sw)[0]) <= (12 if pre else 40)
    # J is ~c * sweeps rotations per column, each within eps of orthogonal
    assert np.abs(J.T @ J - np.eye(c)).max() <= max(1e-13, 1e-15 * c)
    assert np.linalg.norm(BJ @ J.T - B) <= 1e-14 * np.linalg.norm(B) * max(rows, c)
    got = np.sort(sig)[::-1][:k]
    # the exact singular values of the rounded B are s up to the representation error of B
    # (~eps ||B||): relative accuracy for every sigma above ~1e3 eps sigma_max
    big = s > 1e3 * np.finfo(float).eps * s[0]
    assert np.all(np.abs(got[big] - s[big]) <= 1e-8 * s[big] + 1e2 * np.finfo(float).eps * s[0])


@pytest.mark.parametrize("delta", [0.0, 1e-9, 1e-2])
def test_tt_round_accurate_route(tt, delta):
    """tt_round's accurate truncation (QR + cluster Jacobi SVD; automatic for delta / sqrt(d-1)
    < 1e-7, forced at 1e-2 by debug bit 24): on a train whose unfoldings are graded down to
    1e-13, delta = 0 reconstructs to 1e-12 (the Gram route drops everything below ~1e-7), and
    the error bound ||T - round(T)|| <= delta ||T|| holds with ranks equal to the oracle's."""
    from oracle.rounding import tt_round as oracle_round
    rng = np.random.default_rng(91)
    d, N = 6, 4
    x = ttgen.gaussian_tt_vector(rng, N, ttgen.capped_ranks(d, N, 12))
    for k in range(d):
        x[k] = x[k] * np.logspace(0, -13, x[k].shape[2])[None, None, :]
    flags = (1 << 24) if delta >= 1e-7 else 0
    tt.tt_debug_set_flags(flags)
    try:
        out = [h(c) for c in tt.tt_round([g(c) for c in x], delta)]
    finally:
        tt.tt_debug_set_flags(0)
    v, vg = full_vector(x), full_vector(out)
    err = rel_fro(vg, v)
    if delta == 0.0:
        assert err <= 1e-12
    else:
        assert err <= delta * (1 + 1e-6)
        ref = oracle_round(x, delta)
        assert [c.shape for c in out] == [c.shape for c in ref]


# ----------------------------------------------------------------------------------------
# tt_round_async: device-side rank decisions into zero-padded max-rank cores
# ----------------------------------------------------------------------------------------
def _sum_train(a, b):
    d, out = len(a), []
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


def _async_case(case):
    rng = np.random.default_rng(77)
    if case == "random":
        return ttgen.gaussian_tt_vector(rng, 4, [1, 4, 12, 16, 9, 3, 1])
    if case == "sum":       # exactly rank-deficient formal sum T + S + T
        base = ttgen.gaussian_tt_vector(rng, 4, [1, 4, 6, 6, 4, 1])
        x = _sum_train(base, ttgen.gaussian_tt_vector(rng, 4, [1, 3, 5, 5, 3, 1]))
        return _sum_train(x, base)
    if case == "wide":      # bonds wider than their unfoldings: the storage ranks shrink
        return ttgen.gaussian_tt_vector(rng, 2, [1, 5, 9, 20, 7, 1])
    return ttgen.make_inputs(3).x


@pytest.mark.parametrize("case", ["random", "sum", "wide", "config3"])
@pytest.mark.parametrize("delta", [1e-2, 1e-5])
def test_tt_round_async_equals_sync_and_oracle(tt, case, delta):
    """The asynchronous rounding takes the oracle's ranks on the device, its padding is exactly
    zero, the padded train is the rounded tensor as it stands, and the compacted cores agree
    with the synchronous call and the oracle (dense reconstructions)."""
    from oracle.rounding import tt_round as oracle_round
    x = _async_case(case)
    xg = [g(c) for c in x]
    padded, ranks = tt.tt_round_async(xg, delta)
    sync = [h(c) for c in tt.tt_round(xg, delta)]
    ro = [int(v) for v in ranks.tolist()]
    assert ro == [1] + [c.shape[2] for c in sync]
    yo = oracle_round(x, delta)
    assert ro == [1] + [c.shape[2] for c in yo]
    for k, c in enumerate(padded):   # storage ranks chain, padding exactly zero
        assert c.shape[0] >= ro[k] and c.shape[2] >= ro[k + 1]
        if k + 1 < len(padded):
            assert c.shape[2] == padded[k + 1].shape[0]
        ch = h(c)
        assert not ch[ro[k]:, :, :].any() and not ch[:, :, ro[k + 1]:].any()
    comp = [h(c) for c in tt.tt_compact(padded, ranks)]
    assert [c.shape for c in comp] == [c.shape for c in sync]
    v = full_vector(x)
    vp, vc, vs, vo = (full_vector([h(c) for c in padded]), full_vector(comp), full_vector(sync),
                      full_vector(yo))
    assert np.array_equal(vp, vc) or rel_fro(vp, vc) <= 1e-15
    assert rel_fro(vc, vs) <= 1e-10 and rel_fro(vc, vo) <= 1e-10
    assert np.linalg.norm(vc - v) / np.linalg.norm(v) <= delta * (1 + 1e-6)


@pytest.mark.parametrize("case", ["random", "sum", "wide"])
def test_tt_round_async_gram_orthonormalisation(tt, case):
    """Debug bit 29 sends the right-to-left orthonormalisation through the Gram matrix (the
    route of unfoldings too large for one cluster): in the asynchronous call that sweep also
    keeps full-size zero-padded factors and no host read."""
    from oracle.rounding import tt_round as oracle_round
    x = _async_case(case)
    xg = [g(c) for c in x]
    delta = 1e-4
    tt.tt_debug_set_flags(1 << 29)
    try:
        padded, ranks = tt.tt_round_async(xg, delta)
        torch.cuda.synchronize()
    finally:
        tt.tt_debug_set_flags(0)
    yo = oracle_round(x, delta)
    ro = [int(v) for v in ranks.tolist()]
    assert ro == [1] + [c.shape[2] for c in yo]
    for k, c in enumerate(padded):
        ch = h(c)
        assert not ch[ro[k]:, :, :].any() and not ch[:, :, ro[k + 1]:].any()
    comp = [h(c) for c in tt.tt_compact(padded, ranks)]
    v, vc, vo = full_vector(x), full_vector(comp), full_vector(yo)
    assert rel_fro(vc, vo) <= 1e-9          # Gram route on both sweeps: ~eps kappa^2
    assert np.linalg.norm(vc - v) / np.linalg.norm(v) <= delta * (1 + 1e-6)


def test_tt_round_async_max_rank_and_errors(tt):
    rng = np.random.default_rng(78)
    x = [g(c) for c in ttgen.gaussian_tt_vector(rng, 4, [1, 4, 12, 16, 9, 3, 1])]
    padded, ranks = tt.tt_round_async(x, 1e-3, max_rank=5)
    sync = tt.tt_round(x, 1e-3, max_rank=5)
    assert [int(v) for v in ranks.tolist()] == [1] + [c.shape[2] for c in sync]
    assert max(int(v) for v in ranks.tolist()) == 5
    comp = tt.tt_compact(padded, ranks)
    assert rel_fro(full_vector([h(c) for c in comp]), full_vector([h(c) for c in sync])) <= 1e-10
    with pytest.raises(tt.TTError):
        tt.tt_round_async(x, -1.0)


@pytest.mark.parametrize("delta", [0.0, 1e-9, 1e-2])
def test_tt_round_async_accurate_route(tt, delta):
    """Below the Gram floor (delta / sqrt(d-1) < 1e-7, delta = 0 included; forced at 1e-2 by
    debug bit 24) the asynchronous call takes the accurate route too -- cluster QR + cluster
    Jacobi SVD, the singular values ranked and selected on the device: the ranks of the
    synchronous call, exact zero padding, delta = 0 reconstructs the graded train to 1e-12."""
    rng = np.random.default_rng(91)
    d, N = 6, 4
    x = ttgen.gaussian_tt_vector(rng, N, ttgen.capped_ranks(d, N, 12))
    for k in range(d):
        x[k] = x[k] * np.logspace(0, -13, x[k].shape[2])[None, None, :]
    xg = [g(c) for c in x]
    tt.tt_debug_set_flags((1 << 24) if delta >= 1e-7 else 0)
    try:
        sync = [h(c) for c in tt.tt_round(xg, delta)]
        padded, ranks = tt.tt_round_async(xg, delta)
        torch.cuda.synchronize()
    finally:
        tt.tt_debug_set_flags(0)
    ro = [int(v) for v in ranks.tolist()]
    assert ro == [1] + [c.shape[2] for c in sync]
    for k, c in enumerate(padded):
        ch = h(c)
        assert not ch[ro[k]:, :, :].any() and not ch[:, :, ro[k + 1]:].any()
    comp = [h(c) for c in tt.tt_compact(padded, ranks)]
    v, vc, vs = full_vector(x), full_vector(comp), full_vector(sync)
    assert rel_fro(vc, vs) <= 1e-12
    assert rel_fro(vc, v) <= (1e-12 if delta == 0.0 else delta * (1 + 1e-6))


def test_tt_round_async_graph_capture(tt):
    """No host synchronisation inside: the call is captured into a CUDA graph and the replay
    follows new core values in the same buffers."""
    rng = np.random.default_rng(79)
    ranks_in = [1, 4, 10, 12, 6, 1]
    x0 = ttgen.gaussian_tt_vector(rng, 4, ranks_in)
    low = ttgen.gaussian_tt_vector(rng, 4, [1, 2, 3, 3, 2, 1])
    x1 = _sum_train(low, low)                      # rank-deficient: other ranks, same shapes?
    x1 = [np.pad(c, [(0, a.shape[0] - c.shape[0]), (0, 0), (0, a.shape[2] - c.shape[2])])
          for c, a in zip(x1, x0)]
    bufs = [g(c) for c in x0]
    n = [4] * len(bufs)
    ws = torch.empty(tt.tt_round_workspace_size(n, ranks_in), dtype=torch.uint8, device="cuda")
    rk = torch.zeros(len(bufs) + 1, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        tt.tt_round_async(bufs, 1e-4, workspace=ws, stream=s, ranks=rk)   # warm (attributes)
        s.synchronize()
        with torch.cuda.graph(graph, stream=s):
            padded, rk2 = tt.tt_round_async(bufs, 1e-4, workspace=ws, stream=s, ranks=rk)
    for xs in (x1, x0):
        for b, c in zip(bufs, xs):
            b.copy_(g(c))
        graph.replay()
        torch.cuda.synchronize()
        ref = tt.tt_round([g(c) for c in xs], 1e-4)
        assert [int(v) for v in rk.tolist()] == [1] + [c.shape[2] for c in ref]
        comp = tt.tt_compact(padded, rk)
        assert rel_fro(full_vector([h(c) for c in comp]), full_vector([h(c) for c in ref])) <= 1e-10


@pytest.mark.parametrize("direction", ["left", "right"])
def test_orthonormalise_is_asynchronous_and_capturable(tt, direction):
    """With every unfolding on the cluster-QR path nothing is read on the host: the call is
    captured into a CUDA graph and the replay follows new core values, bit-identical to the
    eager call."""
    rng = np.random.default_rng(83)
    ranks = [1, 4, 16, 24, 16, 4, 1]
    x0 = ttgen.gaussian_tt_vector(rng, 4, ranks)
    x1 = ttgen.gaussian_tt_vector(rng, 4, ranks)
    flag = tt.TT_SWEEP_LEFT if direction == "left" else tt.TT_SWEEP_RIGHT
    bufs = [g(c) for c in x0]
    ws = torch.empty(tt.tt_orthonormalise_workspace_size([4] * len(bufs), ranks), dtype=torch.uint8,
                     device="cuda")
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        tt.tt_orthonormalise(bufs, flag, workspace=ws, stream=s)   # warm (attributes)
        s.synchronize()
        with torch.cuda.graph(graph, stream=s):
            out = tt.tt_orthonormalise(bufs, flag, workspace=ws, stream=s)
    for xs in (x1, x0):
        for b, c in zip(bufs, xs):
            b.copy_(g(c))
        graph.replay()
        torch.cuda.synchronize()
        ref = tt.tt_orthonormalise([g(c) for c in xs], flag)
        torch.cuda.synchronize()
        assert [tuple(c.shape) for c in out] == [tuple(c.shape) for c in ref]
        for a, b in zip(out, ref):
            assert torch.equal(a, b)
        assert rel_fro(full_vector([h(c) for c in out]), full_vector(xs)) <= 1e-12


# ----------------------------------------------------------------------------------------
# asynchronous block moves: device-side rank into zero-padded outputs
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("delta", [1e-2, 1e-4, 1e-6])
@pytest.mark.parametrize("m_lt_q", [True, False])
def test_block_move_right_async_equals_sync(tt, delta, m_lt_q):
    rng = np.random.default_rng(91)
    r0, n0, l, r1, n1, r2 = (4, 4, 4, 8, 4, 3) if m_lt_q else (16, 4, 2, 6, 4, 3)
    sig = np.array([3.0, 2.0, 1.0, 0.5, 1e-3, 5e-4, 1e-6, 1e-7])
    Wk_hat = _graded(rng, r0 * n0, l * r1, sig).reshape(r0, n0, l, r1)
    Wk1 = rng.standard_normal((r1, n1, r2))
    Wk_s, W1_s = (h(t) for t in tt.tt_block_move_right(g(Wk_hat), g(Wk1), delta))
    Wk_a, W1_a, rank = tt.tt_block_move_right_async(g(Wk_hat), g(Wk1), delta)
    s = int(rank.item())
    Wk_a, W1_a = h(Wk_a), h(W1_a)
    assert s == Wk_s.shape[2] == block_move_right(Wk_hat, Wk1, delta)[0].shape[2]
    assert Wk_a.shape[2] == min(r0 * n0, l * r1) and W1_a.shape[0] == Wk_a.shape[2]
    assert not Wk_a[:, :, s:].any() and not W1_a[s:].any()      # exact zero padding
    T_s = np.einsum("ais,sjlc->ailjc", Wk_s, W1_s)
    T_a = np.einsum("ais,sjlc->ailjc", Wk_a, W1_a)                # the padded pair as it stands
    assert rel_fro(T_a, T_s) <= 1e-12
    P_a, P_s = Wk_a[:, :, :s].reshape(r0 * n0, s), Wk_s.reshape(r0 * n0, s)
    assert np.abs(P_a @ P_a.T - P_s @ P_s.T).max() <= 1e-12


@pytest.mark.parametrize("delta", [0.0, 1e-3])
@pytest.mark.parametrize("shape", [(2, 4, 5, 4, 3, 6), (8, 4, 32, 4, 4, 8)])
def test_block_move_left_async_equals_sync(tt, shape, delta):
    r0, n0, r1, n1, l, r2 = shape
    rng = np.random.default_rng(92)
    Wkm1 = rng.standard_normal((r0, n0, r1))
    k = min(r1 * l, n1 * r2)
    sig = np.logspace(0, -5, k)
    Wk_hat = _graded(rng, r1 * l, n1 * r2, sig).reshape(r1, l, n1, r2).transpose(0, 2, 1, 3).copy()
    Wh_s, Wk_s = (h(t) for t in tt.tt_block_move_left(g(Wkm1), g(Wk_hat), delta))
    Wh_a, Wk_a, rank = tt.tt_block_move_left_async(g(Wkm1), g(Wk_hat), delta)
    s = int(rank.item())
    Wh_a, Wk_a = h(Wh_a), h(Wk_a)
    assert s == Wk_s.shape[0] == block_move_left(Wkm1, Wk_hat, delta)[1].shape[0]
    assert not Wh_a[..., s:].any() and not Wk_a[s:].any()
    T_s = np.einsum("ails,sjc->ailjc", Wh_s, Wk_s)
    T_a = np.einsum("ails,sjc->ailjc", Wh_a, Wk_a)
    assert rel_fro(T_a, T_s) <= 1e-12


def test_block_move_async_graph_capture(tt):
    """No host read inside: a right move followed by the left move back is one CUDA graph whose
    replay follows new values (the synchronous calls cannot be captured)."""
    rng = np.random.default_rng(93)
    r0, n0, l, r1, n1, r2 = 6, 4, 3, 5, 4, 7
    Wk_hat, Wk1 = g(rng.standard_normal((r0, n0, l, r1))), g(rng.standard_normal((r1, n1, r2)))
    ws = torch.empty(tt.tt_block_move_workspace_size(r0, n0, l, r1, n1, r2), dtype=torch.uint8,
                     device="cuda")
    rk = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        tt.tt_block_move_right_async(Wk_hat, Wk1, 1e-8, workspace=ws, stream=s, rank=rk)   # warm
        s.synchronize()
        with torch.cuda.graph(graph, stream=s):
            Wk, W1, _ = tt.tt_block_move_right_async(Wk_hat, Wk1, 1e-8, workspace=ws, stream=s,
                                                     rank=rk)
    for seed in (1, 2):
        r2g = np.random.default_rng(seed)
        Wk_hat.copy_(g(r2g.standard_normal((r0, n0, l, r1))))
        Wk1.copy_(g(r2g.standard_normal((r1, n1, r2))))
        graph.replay()
        torch.cuda.synchronize()
        T0 = np.einsum("ailb,bjc->ailjc", h(Wk_hat), h(Wk1))
        assert rel_fro(np.einsum("ais,sjlc->ailjc", h(Wk), h(W1)), T0) <= 1e-9
        assert int(rk.item()) == tt.tt_block_move_right(Wk_hat, Wk1, 1e-8)[0].shape[2]
