"""Out-of-bounds write checks (compute-sanitizer is closed on this GPU pool, profiles/r02/
compute_sanitizer_closed.log): every output and the workspace are carved out of a larger buffer
whose guard zones hold a sentinel; after the call the guards must be untouched, the inputs
unchanged (const inputs are never written) and the results equal to the oracle.  Shapes are
ragged (odd extents, rank-1 bonds, extents that are not multiples of any tile) and outputs are
also placed at an 8-byte (not 16-byte) aligned offset, which routes the stage GEMMs through the
unaligned engine."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
SENT = 12345.678
GUARD = 512          # doubles on each side
WGUARD = 1 << 16     # workspace guard bytes
TOL = 1e-11


@pytest.fixture(scope="module")
def tt():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2509_11890_b200 as m
    return m


def guarded(shape, offset=0):
    n = int(np.prod(shape))
    big = torch.full((2 * GUARD + n + offset,), SENT, dtype=torch.float64, device="cuda")
    return big, big[GUARD + offset: GUARD + offset + n].view(*shape)


def check_guards(big, shape, offset=0):
    n = int(np.prod(shape))
    lo, hi = big[: GUARD + offset], big[GUARD + offset + n:]
    assert bool((lo == SENT).all()) and bool((hi == SENT).all()), "write outside the output"


def guarded_ws(nbytes):
    big = torch.full((nbytes + WGUARD,), 0xAB, dtype=torch.uint8, device="cuda")
    return big, big[:nbytes]


def check_ws(big, nbytes):
    assert bool((big[nbytes:] == 0xAB).all()), "write past the workspace size"


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb else float(np.linalg.norm(a))


SHAPES = [(1, 4, 4, 1, 3), (3, 2, 5, 2, 7), (17, 4, 33, 5, 3), (64, 4, 64, 16, 16), (33, 3, 18, 9, 25)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("nvec", [1, 3])
@pytest.mark.parametrize("offset", [0, 1])
def test_matvec_guards(tt, shape, nvec, offset):
    import oracle
    rl, n, rr, Rl, Rr = shape
    rng = np.random.default_rng(rl * 1000 + rr + nvec)
    pl = rng.standard_normal((rl, Rl, rl))
    A = rng.standard_normal((Rl, n, n, Rr))
    pr = rng.standard_normal((rr, Rr, rr))
    X = rng.standard_normal((rl, n, nvec, rr))
    g = lambda a: torch.from_numpy(a).cuda()
    ins = [g(pl), g(A), g(pr), g(X)]
    before = [t.clone() for t in ins]
    bigY, Y = guarded((rl, n, nvec, rr), offset)
    need = tt.tt_local_matvec_workspace_size(rl, n, rr, Rl, Rr, nvec)
    bigW, ws = guarded_ws(need)
    tt.tt_local_matvec_batched(*ins, Y, workspace=ws)
    torch.cuda.synchronize()
    check_guards(bigY, Y.shape, offset)
    check_ws(bigW, need)
    for a, b in zip(ins, before):
        assert torch.equal(a, b)
    assert rel(Y.cpu().numpy(), oracle.local_matvec_batched(pl, A, pr, X)) <= TOL


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("left", [True, False])
def test_interface_guards(tt, shape, left):
    import oracle
    rl, n, rr, Rl, Rr = shape
    rng = np.random.default_rng(rl * 7 + rr)
    x = rng.standard_normal((rl, n, rr))
    A = rng.standard_normal((Rl, n, n, Rr))
    phi = rng.standard_normal((rl, Rl, rl) if left else (rr, Rr, rr))
    g = lambda a: torch.from_numpy(a).cuda()
    ins = [g(phi), g(A), g(x)]
    before = [t.clone() for t in ins]
    oshape = (rr, Rr, rr) if left else (rl, Rl, rl)
    bigO, out = guarded(oshape, 1)
    need = tt.tt_interface_workspace_size(rl, n, rr, Rl, Rr)
    bigW, ws = guarded_ws(need)
    (tt.tt_interface_left if left else tt.tt_interface_right)(*ins, out, workspace=ws)
    torch.cuda.synchronize()
    check_guards(bigO, oshape, 1)
    check_ws(bigW, need)
    for a, b in zip(ins, before):
        assert torch.equal(a, b)
    ref = oracle.interface_left(phi, A, x) if left else oracle.interface_right(phi, A, x)
    assert rel(out.cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("idx", [1, 2])
def test_sweep_w34_and_apply_guards(tt, idx):
    import oracle
    import ttgen
    inp = ttgen.make_inputs(idx)
    x = [torch.from_numpy(c).cuda() for c in inp.x]
    A = [torch.from_numpy(c).cuda() for c in inp.A]
    before = [t.clone() for t in x + A]
    tr = tt._Train(x, A)
    d = len(x)
    pls = [guarded((tr.r[k], tr.R[k], tr.r[k]), k % 2) for k in range(d + 1)]
    prs = [guarded((tr.r[k], tr.R[k], tr.r[k]), (k + 1) % 2) for k in range(d + 1)]
    ys = [guarded(tuple(x[k].shape), k % 2) for k in range(d)]
    need = tt.tt_sweep_w34_workspace_size(tr)
    bigW, ws = guarded_ws(need)
    tt.tt_sweep_w34(x, A, [p[1] for p in pls], [p[1] for p in prs], [y[1] for y in ys], workspace=ws)
    torch.cuda.synchronize()
    for k, (big, t) in enumerate(pls):
        check_guards(big, t.shape, k % 2)
    for k, (big, t) in enumerate(prs):
        check_guards(big, t.shape, (k + 1) % 2)
    for k, (big, t) in enumerate(ys):
        check_guards(big, t.shape, k % 2)
    check_ws(bigW, need)
    oL, oR = oracle.sweep_interfaces(inp.x, inp.A)
    for k in range(d):
        ref = oracle.local_matvec(oL[k], inp.A[k], oR[k + 1], inp.x[k])
        assert rel(ys[k][1].cpu().numpy(), ref) <= TOL
    zs = [guarded((tr.r[k] * tr.R[k], tr.n[k], tr.r[k + 1] * tr.R[k + 1]), k % 2) for k in range(d)]
    tt.tt_operator_apply(x, A, [z[1] for z in zs])
    torch.cuda.synchronize()
    for k, (big, t) in enumerate(zs):
        check_guards(big, t.shape, k % 2)
    for zk, ok in zip(zs, oracle.operator_apply(inp.x, inp.A)):
        assert rel(zk[1].cpu().numpy(), ok) <= TOL
    for a, b in zip(x + A, before):
        assert torch.equal(a, b)


def test_sweep_als_guards(tt):
    import oracle
    import ttgen
    inp = ttgen.make_inputs(2)
    rng = np.random.default_rng(5)
    X = ttgen.random_block(rng, inp.cfg.N, inp.cfg.r, 2)
    x = [torch.from_numpy(c).cuda() for c in inp.x]
    A = [torch.from_numpy(c).cuda() for c in inp.A]
    Xs = [torch.from_numpy(c).cuda() for c in X]
    tr = tt._Train(x, A)
    d = len(x)
    yf = [guarded(tuple(t.shape), k % 2) for k, t in enumerate(Xs)]
    yb = [guarded(tuple(t.shape), (k + 1) % 2) for k, t in enumerate(Xs)]
    pls = [guarded((tr.r[k], tr.R[k], tr.r[k])) for k in range(d + 1)]
    prs = [guarded((tr.r[k], tr.R[k], tr.r[k]), 1) for k in range(d + 1)]
    need = tt.tt_sweep_als_workspace_size(tr, 2)
    bigW, ws = guarded_ws(need)
    tt.tt_sweep_als(x, A, Xs, [y[1] for y in yf], [y[1] for y in yb], [p[1] for p in pls],
                    [p[1] for p in prs], workspace=ws)
    torch.cuda.synchronize()
    for k, (big, t) in enumerate(yf):
        check_guards(big, t.shape, k % 2)
    for k, (big, t) in enumerate(yb):
        check_guards(big, t.shape, (k + 1) % 2)
    for big, t in pls:
        check_guards(big, t.shape, 0)
    for big, t in prs:
        check_guards(big, t.shape, 1)
    check_ws(bigW, need)
    oL, oR = oracle.sweep_interfaces(inp.x, inp.A)
    for k in range(d):
        ref = oracle.local_matvec_batched(oL[k], inp.A[k], oR[k + 1], X[k])
        assert rel(yf[k][1].cpu().numpy(), ref) <= TOL
