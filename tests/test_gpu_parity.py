"""GPU parity: the CUDA path through the C-ABI vs the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star, DESIGN.md §3 A8): relative Frobenius error <= 1e-11 per
output array (each Phi_k, each y_k / Y_k column block, each z_k).  Configs 1-4 are checked
in full; config 5 (full size, the launch configuration bench.py times: tt_sweep_als with
K = 32) on sampled Krylov columns of every core plus every interface, and sampled row slices
of the operator apply.
"""
import concurrent.futures as cf
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL = 1e-11


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def tt():
    _need_gpu()
    import paper_2509_11890_b200 as m
    return m


def g(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def h(t):
    return t.detach().cpu().numpy()


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    if nb == 0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


def test_smoke():
    _need_gpu()
    import __graft_entry__
    __graft_entry__.smoke()


# ----------------------------------------------------------------------------------------
# configs 1-4: full W34 workload (sweep both directions + one matvec per core) + apply
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("idx,engine", [(1, "default"), (2, "default"), (3, "default"),
                                        (4, "default"), (3, "v1"), (4, "v1"), (3, "v2"),
                                        (4, "v2")])
def test_config_w34_parity(tt, idx, engine):
    """engine: default = TMA/mbarrier kernel (v3) where eligible; v1 = the generic
    unaligned-capable kernel for every GEMM; v2 = the cp.async persistent kernel."""
    tt.tt_debug_force_v1(engine == "v1")
    tt.tt_debug_set_variant(1 if engine == "v2" else -1)
    try:
        _w34(tt, idx)
    finally:
        tt.tt_debug_force_v1(False)
        tt.tt_debug_set_variant(-1)


def _w34(tt, idx):
    import oracle
    import ttgen
    inp = ttgen.make_inputs(idx)
    d = inp.cfg.d
    xs, As = [g(c) for c in inp.x], [g(c) for c in inp.A]
    phiL, phiR = tt.tt_sweep_interfaces(xs, As)
    ys = [tt.tt_local_matvec(phiL[k], As[k], phiR[k + 1], xs[k]) for k in range(d)]
    torch.cuda.synchronize()
    oL, oR = oracle.sweep_interfaces(inp.x, inp.A)
    worst = 0.0
    for k in range(d + 1):
        worst = max(worst, rel(h(phiL[k]), oL[k]), rel(h(phiR[k]), oR[k]))
    for k in range(d):
        oy = oracle.local_matvec(oL[k], inp.A[k], oR[k + 1], inp.x[k])
        worst = max(worst, rel(h(ys[k]), oy))
    assert worst <= TOL, worst
    # energy closure on the GPU side: phiL[d] == phiR[0] == <x_k, y_k>
    e = h(phiL[d]).item()
    assert abs(h(phiR[0]).item() - e) <= 1e-12 * abs(e)


@pytest.mark.parametrize("idx", [1, 2, 3, 4])
def test_config_apply_parity(tt, idx):
    import oracle
    import ttgen
    inp = ttgen.make_inputs(idx)
    zs = tt.tt_operator_apply([g(c) for c in inp.x], [g(c) for c in inp.A])
    torch.cuda.synchronize()
    for k in range(inp.cfg.d):
        oz = oracle.apply_core(inp.x[k], inp.A[k])
        gz = h(zs[k])
        zs[k] = None
        assert gz.shape == oz.shape
        assert rel(gz, oz) <= TOL, k


# ----------------------------------------------------------------------------------------
# ragged shapes spanning several tiles in every GEMM stage
# ----------------------------------------------------------------------------------------
RAGGED = [
    # rl, n, rr, Rl, Rr, nvec
    (1, 4, 1, 1, 1, 1),
    (3, 4, 5, 2, 3, 2),
    (37, 4, 53, 7, 11, 5),
    (150, 4, 140, 9, 17, 3),
    (129, 3, 131, 5, 6, 2),        # odd mode size
    (64, 4, 200, 30, 41, 1),       # N*Rr = 164 > 160 -> wide-N tiles in S2
    (257, 2, 33, 3, 2, 4),
]


@pytest.mark.parametrize("shape", RAGGED)
def test_ragged_batched_matvec(tt, shape):
    import oracle
    rl, n, rr, Rl, Rr, nvec = shape
    rng = np.random.default_rng(sum(shape))
    phiL = rng.standard_normal((rl, Rl, rl))
    A = rng.standard_normal((Rl, n, n, Rr))
    phiR = rng.standard_normal((rr, Rr, rr))
    X = rng.standard_normal((rl, n, nvec, rr))
    Y = tt.tt_local_matvec_batched(g(phiL), g(A), g(phiR), g(X))
    ref = oracle.local_matvec_batched(phiL, A, phiR, X)
    for m in range(nvec):
        assert rel(h(Y)[:, :, m, :], ref[:, :, m, :]) <= TOL
    # single-vector entry point == column of the batched one
    y0 = tt.tt_local_matvec(g(phiL), g(A), g(phiR), g(np.ascontiguousarray(X[:, :, 0, :])))
    assert rel(h(y0), ref[:, :, 0, :]) <= TOL


@pytest.mark.parametrize("direct_right", [False, True])
@pytest.mark.parametrize("shape", RAGGED)
def test_ragged_interfaces(tt, shape, direct_right):
    """direct_right: the right update computed directly (debug flag 8) instead of as the
    mirrored left update; both must match the oracle."""
    tt.tt_debug_set_flags(8 if direct_right else 0)
    try:
        _ragged_interfaces(tt, shape)
    finally:
        tt.tt_debug_set_flags(0)


def _ragged_interfaces(tt, shape):
    import oracle
    rl, n, rr, Rl, Rr, _ = shape
    rng = np.random.default_rng(sum(shape) + 1)
    A = rng.standard_normal((Rl, n, n, Rr))
    x = rng.standard_normal((rl, n, rr))
    pl = rng.standard_normal((rl, Rl, rl))
    pr = rng.standard_normal((rr, Rr, rr))
    outL = tt.tt_interface_left(g(pl), g(A), g(x))
    outR = tt.tt_interface_right(g(pr), g(A), g(x))
    assert rel(h(outL), oracle.interface_left(pl, A, x)) <= TOL
    assert rel(h(outR), oracle.interface_right(pr, A, x)) <= TOL


def test_identity_operator_exact(tt):
    """Identity operator and identity interfaces: every product is by 0 or 1, so y == x
    exactly."""
    rng = np.random.default_rng(9)
    for rl, n, rr, nvec in [(1, 4, 1, 1), (40, 4, 130, 3), (256, 4, 256, 2)]:
        X = rng.standard_normal((rl, n, nvec, rr))
        Y = tt.tt_local_matvec_batched(g(np.eye(rl).reshape(rl, 1, rl)),
                                       g(np.eye(n).reshape(1, n, n, 1)),
                                       g(np.eye(rr).reshape(rr, 1, rr)), g(X))
        assert np.array_equal(h(Y), X)


# ----------------------------------------------------------------------------------------
# config 5 at full size, in bench.py's launch configuration
# ----------------------------------------------------------------------------------------
@pytest.mark.timeout(1500)
def test_config5_full_certificate(tt, tmp_path):
    """The complete config-5 parity certificate: every interface, every core,
    all 32 Krylov columns in both sweep directions and the whole unrounded apply output of the
    bench's launch configuration against the oracle as it stands, the oracle's (core, column)
    tasks spread over the host cores (~75 s on the 16-core GPU box; a single core would need
    ~15 min, so smaller hosts keep to the sampled test below)."""
    import json
    import subprocess
    import sys
    if (os.cpu_count() or 1) < 12:
        pytest.skip("fewer than 12 host cores: the sampled config-5 test covers this host")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "config5_certificate.json"
    torch.cuda.empty_cache()
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "config5_certificate.py"),
                        str(out)], cwd=root, capture_output=True, text=True, timeout=1400)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    cert = json.loads(out.read_text())
    assert cert["pass"] is True
    assert max(cert["worst"].values()) <= 1e-11, cert["worst"]


def test_config5_w5_sampled(tt):
    import oracle
    import ttgen
    inp = ttgen.make_inputs(5)
    d, K = inp.cfg.d, inp.cfg.nvec
    xs, As, Xs = [g(c) for c in inp.x], [g(c) for c in inp.A], [g(c) for c in inp.X]
    Yf, Yb, phiL, phiR = tt.tt_sweep_als(xs, As, Xs, Y_bwd=[torch.empty_like(X) for X in Xs])
    torch.cuda.synchronize()
    with cf.ThreadPoolExecutor(2) as ex:   # ctypes releases the GIL: the chains run in parallel
        fl = ex.submit(oracle.sweep_interfaces, inp.x, inp.A, 1)
        fr = ex.submit(oracle.sweep_interfaces, inp.x, inp.A, 2)
        oL = fl.result()[0]
        oR = fr.result()[1]
    # W5 builds phiL[1..d-1] and phiR[1..d-1] (phiL[d], phiR[0] are not needed by a sweep)
    assert h(phiL[0]).item() == 1.0 and h(phiR[d]).item() == 1.0
    for k in range(1, d):
        assert rel(h(phiL[k]), oL[k]) <= TOL, ("phiL", k)
        assert rel(h(phiR[k]), oR[k]) <= TOL, ("phiR", k)
    # Krylov columns: the first, the last and six interior ones drawn from a fixed seed
    rng = np.random.default_rng(20251020)
    cols = sorted({0, K - 1} | set(int(c) for c in rng.choice(np.arange(1, K - 1), 6, replace=False)))
    assert len(cols) == 8
    jobs = {}
    with cf.ThreadPoolExecutor(min(16, os.cpu_count() or 1)) as ex:
        for k in range(d):
            for m in cols:
                xk = np.ascontiguousarray(inp.X[k][:, :, m, :])
                jobs[(k, m)] = ex.submit(oracle.local_matvec, oL[k], inp.A[k], oR[k + 1], xk)
        for (k, m), f in jobs.items():
            ref = f.result()
            assert rel(h(Yf[k][:, :, m, :]), ref) <= TOL, ("fwd", k, m)
            assert rel(h(Yb[k][:, :, m, :]), ref) <= TOL, ("bwd", k, m)
    # forward and backward passes see identical interfaces -> identical results
    for k in range(d):
        assert torch.equal(Yf[k], Yb[k])
    del Yf, Yb, Xs
    torch.cuda.empty_cache()
    zs = tt.tt_operator_apply(xs, As)
    torch.cuda.synchronize()
    for k in [0, 3, 11]:
        rl = inp.x[k].shape[0]
        Rl = inp.A[k].shape[0]
        for a0, a1 in [(0, 1), (rl - 1, rl)]:
            ref = oracle.apply_core(inp.x[k][a0:a1], inp.A[k])
            assert rel(h(zs[k][a0 * Rl:a1 * Rl]), ref) <= TOL, ("apply", k, a0)
    # the whole z of one interior core (2.72 GB), compared in slabs of 32 vector-bond rows
    # (the slab errors combine into the whole core's relative Frobenius error)
    k = 6
    rl, Rl = inp.x[k].shape[0], inp.A[k].shape[0]
    num = den = 0.0
    for a0 in range(0, rl, 32):
        a1 = min(rl, a0 + 32)
        ref = oracle.apply_core(inp.x[k][a0:a1], inp.A[k])
        got = h(zs[k][a0 * Rl:a1 * Rl])
        num += float(np.sum((got - ref) ** 2))
        den += float(np.sum(ref ** 2))
    assert (num / den) ** 0.5 <= TOL, ("apply full core", k, (num / den) ** 0.5)


# ----------------------------------------------------------------------------------------
# graph capture, error paths
# ----------------------------------------------------------------------------------------
def test_graph_capture_equals_eager(tt):
    import ttgen
    inp = ttgen.make_inputs(3)
    xs, As = [g(c) for c in inp.x], [g(c) for c in inp.A]
    eL, eR = tt.tt_sweep_interfaces(xs, As)
    torch.cuda.synchronize()
    gL = tt.alloc_interfaces(xs, As)
    gR = tt.alloc_interfaces(xs, As)
    tr = tt._Train(xs, As)
    ws = torch.empty(tt.tt_sweep_workspace_size(tr), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            tt.tt_sweep_interfaces(xs, As, gL, gR, workspace=ws, stream=s)
    graph.replay()
    torch.cuda.synchronize()
    for a, b in zip(eL + eR, gL + gR):
        assert torch.equal(a, b)


def test_workspace_too_small_enqueues_nothing(tt):
    x = torch.randn(4, 4, 4, dtype=torch.float64, device="cuda")
    A = torch.randn(2, 4, 4, 2, dtype=torch.float64, device="cuda")
    pl = torch.randn(4, 2, 4, dtype=torch.float64, device="cuda")
    pr = torch.randn(4, 2, 4, dtype=torch.float64, device="cuda")
    y = torch.full_like(x, 7.0)
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(tt.TTError) as ei:
        tt.tt_local_matvec(pl, A, pr, x, y, workspace=ws)
    assert ei.value.status == 4
    torch.cuda.synchronize()
    assert bool((y == 7.0).all())
    with pytest.raises(TypeError):
        tt.tt_local_matvec(pl.cpu(), A, pr, x)


# ----------------------------------------------------------------------------------------
# more paths: small W5 sweeps, d = 1, rectangular apply, sweep graph capture, errors
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("with_bwd", [True, False])
def test_sweep_als_small_vs_oracle(tt, with_bwd):
    """tt_sweep_als (W5) on config-3 shapes with a 3-column block, both passes vs oracle."""
    import oracle
    import ttgen
    inp = ttgen.make_inputs(3)
    d = inp.cfg.d
    rng = np.random.default_rng(33)
    X = ttgen.random_block(rng, inp.cfg.N, inp.cfg.r, 3)
    xs, As, Xs = [g(c) for c in inp.x], [g(c) for c in inp.A], [g(c) for c in X]
    Yb = [torch.empty_like(t) for t in Xs] if with_bwd else None
    Yf, Yb, phiL, phiR = tt.tt_sweep_als(xs, As, Xs, Y_bwd=Yb)
    torch.cuda.synchronize()
    oL, oR = oracle.sweep_interfaces(inp.x, inp.A)
    for k in range(1, d):
        assert rel(h(phiL[k]), oL[k]) <= TOL and rel(h(phiR[k]), oR[k]) <= TOL
    for k in range(d):
        ref = oracle.local_matvec_batched(oL[k], inp.A[k], oR[k + 1], X[k])
        assert rel(h(Yf[k]), ref) <= TOL
        if with_bwd:
            assert torch.equal(Yf[k], Yb[k])


def test_single_core_train(tt):
    """d = 1: the interfaces are the boundary values and phiL[1] = phiR[0] = x^T A x."""
    import oracle
    rng = np.random.default_rng(5)
    x = rng.standard_normal((1, 6, 1))
    A = rng.standard_normal((1, 6, 6, 1))
    pl, pr = tt.tt_sweep_interfaces([g(x)], [g(A)])
    oL, oR = oracle.sweep_interfaces([x], [A])
    assert rel(h(pl[1]), oL[1]) <= TOL and rel(h(pr[0]), oR[0]) <= TOL
    z = tt.tt_operator_apply([g(x)], [g(A)])
    assert rel(h(z[0]), oracle.apply_core(x, A)) <= TOL


@pytest.mark.parametrize("shapes,rs", [
    ([(1, 5, 3, 2), (2, 2, 3, 4), (4, 4, 3, 1)], [1, 3, 9, 1]),       # small: shared-memory kernel
    ([(1, 3, 3, 30), (30, 2, 3, 20), (20, 5, 3, 1)], [1, 16, 24, 1]),  # r R >= 256: register kernel
])
def test_rectangular_apply(tt, shapes, rs):
    import oracle
    rng = np.random.default_rng(71)
    x = [rng.standard_normal((rs[k], shapes[k][2], rs[k + 1])) for k in range(3)]
    A = [rng.standard_normal(s) for s in shapes]
    z = tt.tt_operator_apply([g(c) for c in x], [g(c) for c in A])
    for k in range(3):
        assert rel(h(z[k]), oracle.apply_core(x[k], A[k])) <= TOL


def test_sweep_als_graph_capture_equals_eager(tt):
    """The W5 sweep forks a side stream internally; it must capture into one CUDA graph."""
    import ttgen
    inp = ttgen.make_inputs(3)
    rng = np.random.default_rng(44)
    X = ttgen.random_block(rng, inp.cfg.N, inp.cfg.r, 2)
    xs, As, Xs = [g(c) for c in inp.x], [g(c) for c in inp.A], [g(c) for c in X]
    Ye, _, pLe, pRe = tt.tt_sweep_als(xs, As, Xs)
    torch.cuda.synchronize()
    tr = tt._Train(xs, As)
    ws = torch.empty(tt.tt_sweep_als_workspace_size(tr, 2), dtype=torch.uint8, device="cuda")
    Yg = [torch.zeros_like(t) for t in Xs]
    pLg, pRg = tt.alloc_interfaces(xs, As), tt.alloc_interfaces(xs, As)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            tt.tt_sweep_als(xs, As, Xs, Yg, None, pLg, pRg, workspace=ws, stream=s)
    graph.replay()
    torch.cuda.synchronize()
    for a, b in zip(Ye + pLe[:-1] + pRe[1:], Yg + pLg[:-1] + pRg[1:]):
        assert torch.equal(a, b)


def test_sweep_workspace_errors(tt):
    import ttgen
    inp = ttgen.make_inputs(1)
    xs, As = [g(c) for c in inp.x], [g(c) for c in inp.A]
    small = torch.empty(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(tt.TTError) as ei:
        tt.tt_sweep_interfaces(xs, As, workspace=small)
    assert ei.value.status == 4
    with pytest.raises(tt.TTError) as ei:   # aliasing: output interface == input core
        pl = tt.alloc_interfaces(xs, As)
        pl[2] = xs[1]
        tt.tt_sweep_interfaces(xs, As, phiL=pl, directions=tt.TT_SWEEP_LEFT)
    assert ei.value.status in (3, 1)


# ----------------------------------------------------------------------------------------
# matrix-free local GMRES vs the oracle GMRES
# ----------------------------------------------------------------------------------------
def _mixed_canonical_system(idx, k, seed=3):
    import oracle
    import ttgen
    inp = ttgen.make_inputs(idx)
    xl = ttgen.left_orthonormalise(inp.x)
    xr = ttgen.right_orthonormalise(inp.x)
    mixed = xl[:k] + [inp.x[k]] + xr[k + 1:]
    pl, _ = oracle.sweep_interfaces(mixed, inp.A, 1)
    _, pr = oracle.sweep_interfaces(mixed, inp.A, 2)
    return mixed, inp.A, pl[k], pr[k + 1], np.random.default_rng(seed)


@pytest.mark.parametrize("idx,k,K,m,cycles,kaug", [(2, 3, 4, 12, 2, 0), (4, 5, 3, 8, 1, 0),
                                                  (3, 1, 5, 10, 2, 0), (2, 3, 4, 5, 4, 2),
                                                  (3, 5, 3, 6, 3, 1),
                                                  # K = 1: the fused cluster orthogonalisation
                                                  (3, 5, 1, 10, 2, 0), (2, 3, 1, 12, 3, 2),
                                                  (4, 6, 1, 8, 2, 0), (2, 0, 1, 6, 2, 0)])
def test_local_gmres_vs_oracle(tt, idx, k, K, m, cycles, kaug):
    """Fixed m, cycles (and augmentation k for LGMRES) and tol = 0 on both sides: the
    iterates must agree (<= 1e-11) and take the same number of Arnoldi steps."""
    from oracle.gmres import local_gmres_batched
    mixed, A, phiL, phiR, rng = _mixed_canonical_system(idx, k)
    rl, n, rr = mixed[k].shape
    F = rng.standard_normal((rl, n, K, rr))
    X0 = 0.1 * rng.standard_normal((rl, n, K, rr))
    Xo, relo, itso = local_gmres_batched(phiL, A[k], phiR, F, X0, m=m, cycles=cycles, tol=0.0,
                                         k=kaug)
    Xg, relg, itsg = tt.tt_local_gmres(g(phiL), g(A[k]), g(phiR), g(F), g(X0.copy()), m=m,
                                       cycles=cycles, tol=0.0, k_aug=kaug)
    torch.cuda.synchronize()
    for j in range(K):
        assert rel(h(Xg)[:, :, j, :], Xo[:, :, j, :]) <= TOL, j
    assert (h(itsg) == itso).all()
    assert np.allclose(h(relg), relo, rtol=1e-6, atol=1e-14)


def test_local_gmres_converges_to_dense_solution(tt):
    """SPD Kronecker-sum operator, orthonormal frame (config-2 core 3): GMRES to tol 1e-13
    reproduces the dense solve of the projected system."""
    from dense_ref import full_matrix, projected_operator
    mixed, A, phiL, phiR, rng = _mixed_canonical_system(2, 2)
    rl, n, rr = mixed[2].shape
    F = rng.standard_normal((rl, n, 2, rr))
    Xg, relg, itsg = tt.tt_local_gmres(g(phiL), g(A[2]), g(phiR), g(F), m=30, cycles=4,
                                       tol=1e-13)
    torch.cuda.synchronize()
    L = projected_operator(mixed, full_matrix(A), 2)
    for j in range(2):
        ref = np.linalg.solve(L, F[:, :, j, :].ravel())
        assert rel(h(Xg)[:, :, j, :].ravel(), ref) <= 1e-11
    assert (h(relg) <= 1e-13).all()


@pytest.mark.parametrize("idx,k,m,kaug", [(3, 5, 10, 0), (4, 6, 12, 2)])
def test_local_gmres_fused_orth_equals_separate_kernels(tt, idx, k, m, kaug):
    """K = 1: the one-launch cluster orthogonalisation step (CGS2 + Givens + scaling) against the
    separate kernels (debug flag 1 << 26): same Arnoldi step counts, iterates within rounding."""
    mixed, A, phiL, phiR, rng = _mixed_canonical_system(idx, k)
    rl, n, rr = mixed[k].shape
    F = rng.standard_normal((rl, n, 1, rr))
    out = []
    for flags in (0, 1 << 26):
        tt.tt_debug_set_flags(flags)
        try:
            out.append(tt.tt_local_gmres(g(phiL), g(A[k]), g(phiR), g(F), m=m, cycles=3, tol=1e-12,
                                         k_aug=kaug))
            torch.cuda.synchronize()
        finally:
            tt.tt_debug_set_flags(0)
    (Xa, ra, ia), (Xb, rb, ib) = out
    assert (h(ia) == h(ib)).all()
    assert rel(h(Xa), h(Xb)) <= 1e-11
    assert np.allclose(h(ra), h(rb), rtol=1e-6, atol=1e-14)


@pytest.mark.parametrize("idx", [1, 2, 3, 4])
def test_small_boundary_runs_equal_stage_gemms(tt, idx):
    """Runs of small boundary updates in one fused CTA (default) against the three DMMA stage
    GEMMs per core (debug bit 28): interfaces and W34 matvecs agree to rounding."""
    import ttgen
    inp = ttgen.make_inputs(idx)
    x = [g(c) for c in inp.x]
    A = [g(c) for c in inp.A]
    outs = []
    for flags in (0, 1 << 28):
        tt.tt_debug_set_flags(flags)
        try:
            pl, pr = tt.tt_sweep_interfaces(x, A)
            y, ql, qr = tt.tt_sweep_w34(x, A)
            torch.cuda.synchronize()
            outs.append(pl + pr + y + ql + qr)
        finally:
            tt.tt_debug_set_flags(0)
    for a, b in zip(*outs):
        assert rel(h(a), h(b)) <= 1e-13


def test_local_gmres_errors(tt):
    F = torch.zeros(2, 4, 65, 2, dtype=torch.float64, device="cuda")
    A = torch.zeros(1, 4, 4, 1, dtype=torch.float64, device="cuda")
    P = torch.zeros(2, 1, 2, dtype=torch.float64, device="cuda")
    with pytest.raises(tt.TTError) as ei:
        tt.tt_local_gmres(P, A, P, F, m=4)
    assert ei.value.status == 1
    F = torch.zeros(2, 4, 3, 2, dtype=torch.float64, device="cuda")
    X, rr_, it = tt.tt_local_gmres(P, A, P, F, m=4, cycles=2, tol=1e-12)   # zero rhs -> zero
    torch.cuda.synchronize()
    assert not h(X).any() and (h(it) == 0).all()


# ----------------------------------------------------------------------------------------
# two-site (DMRG supercore) local matvec vs the oracle
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("shape", [
    # rl, n1, n2, rr, Rl, Rm, Rr, nvec
    (3, 2, 2, 5, 2, 3, 2, 1),
    (37, 2, 2, 45, 6, 9, 5, 3),
    (64, 2, 3, 40, 16, 12, 8, 2),
    (128, 2, 2, 128, 25, 25, 25, 4),
])
def test_two_site_matvec_vs_oracle(tt, shape):
    import oracle
    rl, n1, n2, rr, Rl, Rm, Rr, nvec = shape
    rng = np.random.default_rng(sum(shape))
    phiL = rng.standard_normal((rl, Rl, rl))
    A1 = rng.standard_normal((Rl, n1, n1, Rm))
    A2 = rng.standard_normal((Rm, n2, n2, Rr))
    phiR = rng.standard_normal((rr, Rr, rr))
    W = rng.standard_normal((rl, n1, n2, nvec, rr))
    Y = tt.tt_local_matvec_two_site(g(phiL), g(A1), g(A2), g(phiR), g(W))
    torch.cuda.synchronize()
    for m in range(nvec):
        ref = oracle.local_matvec_two_site(phiL, A1, A2, phiR, np.ascontiguousarray(W[:, :, :, m, :]))
        assert rel(h(Y)[:, :, :, m, :], ref) <= TOL, m


# ----------------------------------------------------------------------------------------
# projected KKT block system action vs the oracle
# ----------------------------------------------------------------------------------------
KKT_TERMS = [(0, 0, 0, -1, -1.0), (0, 1, 1, -1, 1.0), (1, 0, 2, -1, -1.0), (1, 2, 3, -1, 1.0),
             (2, 0, 4, -1, 1.0), (2, 1, 5, 6, 1.0), (2, 2, 5, 7, 1.0)]


@pytest.mark.parametrize("rl,n,rr,Rmax", [(5, 4, 7, 3), (64, 4, 96, 16), (129, 4, 128, 25)])
def test_block_local_matvec_vs_oracle(tt, rl, n, rr, Rmax):
    import oracle
    rng = np.random.default_rng(rl + rr)
    ops_h, ops_d = [], []
    for o in range(8):
        Rl_, Rr_ = int(rng.integers(1, Rmax + 1)), int(rng.integers(1, Rmax + 1))
        op = (rng.standard_normal((rl, Rl_, rl)), rng.standard_normal((Rl_, n, n, Rr_)),
              rng.standard_normal((rr, Rr_, rr)))
        ops_h.append(op)
        ops_d.append(tuple(g(a) for a in op))
    X = rng.standard_normal((rl, n, 3, rr))
    Y = tt.tt_block_local_matvec(ops_d, KKT_TERMS, g(X))
    torch.cuda.synchronize()
    ref = oracle.block_local_matvec(ops_h, KKT_TERMS, X)
    for b in range(3):
        assert rel(h(Y)[:, :, b, :], ref[:, :, b, :]) <= TOL, b


# ----------------------------------------------------------------------------------------
# TT rounding vs the oracle (Oseledets Alg. 2)
# ----------------------------------------------------------------------------------------
def _tt_sum(a, b, sb=1.0):
    d = len(a)
    out = []
    for k in range(d):
        ca, cb = a[k], (sb * b[k] if k == 0 else b[k])
        if d == 1:
            out.append(ca + cb)
        elif k == 0:
            out.append(np.concatenate([ca, cb], axis=2))
        elif k == d - 1:
            out.append(np.concatenate([ca, cb], axis=0))
        else:
            c = np.zeros((ca.shape[0] + cb.shape[0], ca.shape[1], ca.shape[2] + cb.shape[2]))
            c[:ca.shape[0], :, :ca.shape[2]] = ca
            c[ca.shape[0]:, :, ca.shape[2]:] = cb
            out.append(c)
    return out


@pytest.mark.parametrize("case", ["random", "sum", "config3"])
@pytest.mark.parametrize("delta", [1e-2, 1e-6])
def test_tt_round_vs_oracle(tt, case, delta):
    import ttgen
    from oracle.rounding import tt_round as oracle_round
    rng = np.random.default_rng(5)
    if case == "random":
        x = ttgen.gaussian_tt_vector(rng, 4, [1, 4, 12, 16, 9, 3, 1])
    elif case == "sum":
        base = ttgen.gaussian_tt_vector(rng, 4, [1, 4, 6, 6, 4, 1])
        x = _tt_sum(base, ttgen.gaussian_tt_vector(rng, 4, [1, 3, 5, 5, 3, 1]))
        x = _tt_sum(x, base)                       # exactly rank-deficient formal sum
    else:
        x = ttgen.make_inputs(3).x
    from dense_ref import full_vector
    yo = oracle_round(x, delta)
    yg = [h(c) for c in tt.tt_round([g(c) for c in x], delta)]
    assert [c.shape for c in yg] == [c.shape for c in yo]
    # dense reconstructions (config 3: 4^10 entries); a TT inner-product difference would
    # cancel catastrophically at this accuracy
    v, vo, vg = full_vector(x), full_vector(yo), full_vector(yg)
    assert rel(vg, vo) <= TOL
    assert np.linalg.norm(vg - v) / np.linalg.norm(v) <= delta * (1 + 1e-6)


@pytest.mark.parametrize("n", [1, 2, 7, 64, 65, 129, 256, 300, 1024])
def test_jacobi_eigen_vs_numpy(tt, n):
    rng = np.random.default_rng(n)
    M = rng.standard_normal((n, n))
    G = M @ M.T
    lam, V = tt.tt_debug_sym_eigen(g(G))
    torch.cuda.synchronize()
    ref = np.linalg.eigvalsh(G)[::-1]
    assert np.allclose(h(lam), ref, rtol=1e-12, atol=1e-12 * ref[0])
    Vh = h(V)
    assert np.allclose(Vh.T @ Vh, np.eye(n), atol=1e-12)
    assert np.allclose(G @ Vh, Vh * h(lam), atol=1e-10 * ref[0])


def test_block_and_elementwise_jacobi_agree(tt):
    """The block-Jacobi kernel (n > 64) and the element-wise kernel (debug flag 256) give the
    same spectrum, including exactly repeated and zero eigenvalues."""
    rng = np.random.default_rng(9)
    Q = np.linalg.qr(rng.standard_normal((200, 200)))[0]
    lamv = np.concatenate([np.repeat([5.0, 2.0], 40), rng.uniform(0.1, 1.0, 100), np.zeros(20)])
    G = (Q * lamv) @ Q.T
    lb, Vb = tt.tt_debug_sym_eigen(g(G))
    tt.tt_debug_set_flags(256)
    le, Ve = tt.tt_debug_sym_eigen(g(G))
    tt.tt_debug_set_flags(0)
    torch.cuda.synchronize()
    ref = np.sort(lamv)[::-1]
    assert np.allclose(h(lb), ref, atol=1e-12 * 5) and np.allclose(h(le), ref, atol=1e-12 * 5)
    for V, lam in ((h(Vb), h(lb)), (h(Ve), h(le))):
        assert np.allclose(V.T @ V, np.eye(200), atol=1e-12)
        assert np.allclose(G @ V, V * lam, atol=1e-10 * 5)


@pytest.mark.parametrize("flags", [0, 1 << 2, 1 << 16])
@pytest.mark.parametrize("n", [24, 33, 64, 100, 256])
def test_block_jacobi_kernels_agree_with_lapack(tt, n, flags):
    """Every block-Jacobi kernel (default: cross-pair inner sweeps + two-rsqrt rotations + DMMA
    updates, blocks of 16; bit 2: blocks of 32; bit 16: the first kernel) against LAPACK on a
    Gram matrix graded over 12 decades, including sizes that pad (33, 100)."""
    rng = np.random.default_rng(1000 + n)
    Q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    lamv = np.logspace(0, -12, n)
    G = (Q * lamv) @ Q.T
    G = (G + G.T) / 2
    tt.tt_debug_set_flags(flags)
    try:
        lam, V = tt.tt_debug_sym_eigen(g(G))
        torch.cuda.synchronize()
    finally:
        tt.tt_debug_set_flags(0)
    ref = np.linalg.eigvalsh(G)[::-1]
    assert np.allclose(h(lam), ref, rtol=0, atol=8 * n * 2.2e-16)   # both sides err ~ n eps
    Vh = h(V)
    assert np.abs(Vh.T @ Vh - np.eye(n)).max() <= 1e-12
    assert np.abs(G @ Vh - Vh * h(lam)).max() <= 1e-13


@pytest.mark.parametrize("scale", [1e-60, 1.0, 1e60])
def test_block_jacobi_scale_invariance(tt, scale):
    """The rotations are computed from power-of-two-scaled entries: the eigenvectors of s G are
    those of G and the eigenvalues scale, for s far from 1 (|s G|^2 still representable)."""
    rng = np.random.default_rng(77)
    n = 96
    M = rng.standard_normal((3 * n, n))
    G = M.T @ M
    lam1, V1 = tt.tt_debug_sym_eigen(g(G))
    lams, Vs = tt.tt_debug_sym_eigen(g(G * scale))
    torch.cuda.synchronize()
    assert np.allclose(h(lams) / scale, h(lam1), rtol=1e-13)
    Vh = h(Vs)
    assert np.abs(Vh.T @ Vh - np.eye(n)).max() <= 1e-12
    assert np.abs((G * scale) @ Vh - Vh * h(lams)).max() <= 1e-12 * scale * h(lam1)[0]


# ----------------------------------------------------------------------------------------
# W34 as one DAG-scheduled call (tt_sweep_w34)
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("flags,dag", [(0, 0), (8388608, 0), (0, 1), (0, 2)])
@pytest.mark.parametrize("idx", [1, 2, 3, 4])
def test_sweep_w34_call_vs_oracle_and_separate_calls(tt, idx, flags, dag):
    """dag 0: the stream/event version (T2 reuse, or bit 23: three-stage matvecs); dag 1 / 2:
    the experimental persistent DAG executor (4- / 8-warp tiles)."""
    import oracle
    import ttgen
    inp = ttgen.make_inputs(idx)
    x = [g(c) for c in inp.x]
    A = [g(c) for c in inp.A]
    tt.tt_debug_set_flags(flags)
    tt.tt_debug_set_dag(dag)
    try:
        y, pl, pr = tt.tt_sweep_w34(x, A)
        torch.cuda.synchronize()
        y_b, pl_b, pr_b = tt.tt_sweep_w34(x, A)   # repeat call: counters re-zeroed, same result
        torch.cuda.synchronize()
    finally:
        tt.tt_debug_set_flags(0)
        tt.tt_debug_set_dag(0)
    for a, b in zip(y + pl + pr, y_b + pl_b + pr_b):
        assert torch.equal(a, b)   # deterministic (split-K partials summed in split order)
    # the separate calls: identical for the stream version (same kernels), within a few ulps
    # of accumulated rounding for the DAG executor (other tiles and split-K factors)
    pl2, pr2 = tt.alloc_interfaces(x, A), tt.alloc_interfaces(x, A)
    tt.tt_sweep_interfaces(x, A, pl2, pr2)
    for k in range(len(x)):
        y2 = tt.tt_local_matvec(pl2[k], A[k], pr2[k + 1], x[k])
        # boundary cores: W34 reuses the fused small update's stage-2 intermediate (FMA loops)
        # where tt_local_matvec runs the DMMA stages -> equal up to rounding order
        assert rel(h(y[k]), h(y2)) <= 1e-13
    for a, b in zip(pl + pr, pl2 + pr2):
        if dag == 0:
            assert torch.equal(a, b)
        else:
            assert rel(h(a), h(b)) <= 1e-13
    # and the oracle
    opl, opr = oracle.sweep_interfaces(inp.x, inp.A, 3)
    for k in range(len(x)):
        ref = oracle.local_matvec(opl[k], inp.A[k], opr[k + 1], inp.x[k])
        assert rel(h(y[k]), ref) <= TOL
        assert rel(h(pl[k + 1]), opl[k + 1]) <= TOL and rel(h(pr[k]), opr[k]) <= TOL


def test_sweep_w34_graph_capture(tt):
    import ttgen
    inp = ttgen.make_inputs(3)
    x = [g(c) for c in inp.x]
    A = [g(c) for c in inp.A]
    y0, _, _ = tt.tt_sweep_w34(x, A)
    torch.cuda.synchronize()
    pl, pr = tt.alloc_interfaces(x, A), tt.alloc_interfaces(x, A)
    y = [torch.zeros_like(c) for c in x]
    tr = tt._Train(x, A)
    ws = torch.empty(tt.tt_sweep_w34_workspace_size(tr), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            tt.tt_sweep_w34(x, A, pl, pr, y, workspace=ws, stream=s)
    graph.replay()
    torch.cuda.synchronize()
    for a, b in zip(y, y0):
        assert torch.equal(a, b)


def test_local_gmres_converged_cycle_is_gated(tt):
    """Once every column has converged, the rest of the cycle's Arnoldi steps are device-gated
    no-ops: a solve that converges early costs far less than the same launch sequence with
    tol = 0, and its result equals the oracle's."""
    from oracle.gmres import local_gmres_batched
    mixed, A, phiL, phiR, rng = _mixed_canonical_system(2, 3)
    k = 3
    shape = mixed[k].shape
    F = rng.standard_normal((shape[0], shape[1], 4, shape[2]))
    args = (g(phiL), g(A[k]), g(phiR), g(F))

    def run(tol):
        X = torch.zeros_like(args[3])
        tt.tt_local_gmres(*args, X, m=60, cycles=1, tol=tol)   # warm
        X.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = tt.tt_local_gmres(*args, X, m=60, cycles=1, tol=tol)
        e1.record()
        torch.cuda.synchronize()
        return out, e0.elapsed_time(e1)
    (X1, rel1, it1), t_conv = run(1e-8)
    (_, _, it0), t_full = run(0.0)
    assert int(h(it1).max()) < 60 and int(h(it0).min()) == 60
    assert t_conv < 0.8 * t_full
    Xo, relo, ito = local_gmres_batched(phiL, A[k], phiR, F, np.zeros_like(F), m=60, cycles=1,
                                        tol=1e-8)
    assert np.array_equal(h(it1), ito)
    assert rel(h(X1), Xo) <= 1e-9


# Every tile configuration of the v3 engine the latency policy (or a probe) can select, with
# forced split-K factors that leave ragged K ranges (KT = 25 k-tiles split 3 / 8 / 16 ways):
# interface update + single-vector matvec vs the oracle.  Guards the 4-warp / 4-CTA-per-SM
# configurations and the no-empty-split clamp of the split-K planner.
@pytest.mark.timeout(120)
@pytest.mark.parametrize("cfg", list(range(10, 23)) + [24, 26, 27])
@pytest.mark.parametrize("ks", [1, 3, 8, 16])
def test_forced_tile_configs(tt, cfg, ks):
    import oracle
    rl, n, rr, Rl, Rr = 100, 4, 36, 5, 7     # S1 K = 100, S3' K = rl*n = 400 (25 k-tiles)
    rng = np.random.default_rng(cfg * 100 + ks)
    phiL = rng.standard_normal((rl, Rl, rl))
    A = rng.standard_normal((Rl, n, n, Rr))
    phiR = rng.standard_normal((rr, Rr, rr))
    x = rng.standard_normal((rl, n, rr))
    tt.tt_debug_set_variant(cfg + 100 * ks)
    try:
        out = tt.tt_interface_left(g(phiL), g(A), g(x))
        y = tt.tt_local_matvec(g(phiL), g(A), g(phiR), g(x))
        torch.cuda.synchronize()
    finally:
        tt.tt_debug_set_variant(-1)
    assert rel(h(out), oracle.interface_left(phiL, A, x)) <= TOL
    assert rel(h(y), oracle.local_matvec(phiL, A, phiR, x)) <= TOL


@pytest.mark.timeout(300)
@pytest.mark.parametrize("idx", [3, 4])
def test_latency_policy_w34_vs_default_policy(tt, idx):
    """The small-GEMM latency policy (tile + split-K model) against the default tile policy
    (debug flag 8192) on the config-3/4 W34 DAG: same interfaces and matvecs (<= 1e-11)."""
    import ttgen
    inp = ttgen.make_inputs(idx)
    x = [g(c) for c in inp.x]
    A = [g(c) for c in inp.A]
    outs = []
    for flags in (0, 8192):
        tt.tt_debug_set_flags(flags)
        try:
            pl, pr = tt.alloc_interfaces(x, A), tt.alloc_interfaces(x, A)
            y = [torch.empty_like(c) for c in x]
            tr = tt._Train(x, A)
            ws = torch.empty(tt.tt_sweep_w34_workspace_size(tr), dtype=torch.uint8, device="cuda")
            tt.tt_sweep_w34(x, A, pl, pr, y, workspace=ws)
            torch.cuda.synchronize()
        finally:
            tt.tt_debug_set_flags(0)
        outs.append([h(t) for t in pl + pr + y])
    for a, b in zip(*outs):
        assert rel(a, b) <= TOL


# Operator-core stage with the resident-B GEMM variant (debug bit 25: the whole A-hat loaded
# once per CTA, the ring carries only T1 tiles) and with the ring (default), at a size above
# the small-GEMM latency path (S2 = 2 x 262144 x 144 x 144 = 10.9 GFLOP > 10 GFLOP) with a
# ragged last tile.
@pytest.mark.timeout(300)
@pytest.mark.parametrize("flags", [0, 33554432 | 8192])   # bit 13 (8192): no latency policy, so
@pytest.mark.parametrize("shape", [(64, 4, 64, 36, 36, 64), (60, 4, 68, 25, 36, 88)])   # B_RES runs
def test_operator_core_stage_resident_b(tt, shape, flags):
    import oracle
    rl, n, rr, Rl, Rr, nvec = shape
    rng = np.random.default_rng(sum(shape) + flags % 7)
    phiL = rng.standard_normal((rl, Rl, rl))
    A = rng.standard_normal((Rl, n, n, Rr))
    phiR = rng.standard_normal((rr, Rr, rr))
    X = rng.standard_normal((rl, n, nvec, rr))
    tt.tt_debug_set_flags(flags)
    try:
        Y = tt.tt_local_matvec_batched(g(phiL), g(A), g(phiR), g(X))
        torch.cuda.synchronize()
    finally:
        tt.tt_debug_set_flags(0)
    ref = oracle.local_matvec_batched(phiL, A, phiR, X)
    for m in range(nvec):
        assert rel(h(Y)[:, :, m, :], ref[:, :, m, :]) <= TOL


@pytest.mark.parametrize("idx", [1, 3, 5])
def test_apply_register_blocked_path(tt, idx):
    """The register-blocked apply kernel (debug bit 27) against the default row-block kernel and
    the oracle (config 5: cores 0-3 and 11 in full, which cover both kernels' boundary cases)."""
    import oracle
    import ttgen
    inp = ttgen.make_inputs(idx)
    x = [g(c) for c in inp.x]
    A = [g(c) for c in inp.A]
    ks = range(len(x)) if idx != 5 else [0, 1, 2, 3, len(x) - 1]
    zd = tt.tt_operator_apply(x, A)
    tt.tt_debug_set_flags(1 << 27)
    try:
        zr = tt.tt_operator_apply(x, A)
        torch.cuda.synchronize()
    finally:
        tt.tt_debug_set_flags(0)
    for k in ks:
        assert torch.equal(zd[k], zr[k])   # same FMA order per output: bit-identical
        assert rel(h(zr[k]), oracle.apply_core(inp.x[k], inp.A[k])) <= TOL
