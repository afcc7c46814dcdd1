"""GPU parity of the fused S1 -> S2 matvec kernel (csrc/tt_fused12.cuh: the first intermediate
of the three-product local matvec, stays in shared memory) against the CPU oracle
and against the three-stage path, on shapes that exercise every edge of the fused tile:
ragged groups of four left-bond indices, operator bonds below the 36-row tile, k-tile padding
in both phases, one and several Krylov columns, several units per CTA.

Bar: relative Frobenius error <= 1e-11 per Krylov column (BASELINE.json north_star)."""
import numpy as np
import pytest

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


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb else 1.0))


FUSED_SHAPES = [
    # rl, rr, Rl, Rr, nvec     (n = 4; rr % 16 == 0, rl even, Rr % 4 == 0: the fused preconditions)
    (8, 16, 36, 36, 3),        # the config-5 operator bonds, two groups of a'
    (6, 16, 36, 36, 1),        # ragged last group (a' = 4, 5 only)
    (2, 32, 5, 4, 2),          # odd al: phase-2 k-tile padding (20 of 32 k-rows), 16 columns
    (34, 48, 7, 12, 2),        # phase-1 k-tile padding (34 of 48), ragged group, 3 b tiles
    (64, 64, 16, 16, 4),       # config-3 interior core
    (36, 16, 36, 8, 1),
    (128, 128, 25, 24, 2),     # several units per CTA (32 x 8 x 2 = 512 units on 148 CTAs)
    (40, 80, 1, 4, 5),         # al = 1
]


@pytest.mark.parametrize("mode", [1, 2, 3, 5, 8, 98, 99, 194])
@pytest.mark.parametrize("shape", FUSED_SHAPES)
def test_fused_matvec_vs_oracle(tt, shape, mode):
    import oracle
    rl, rr, Rl, Rr, nvec = shape
    rng = np.random.default_rng(sum(shape) + 7)
    phiL = rng.standard_normal((rl, Rl, rl))
    A = rng.standard_normal((Rl, 4, 4, Rr))
    phiR = rng.standard_normal((rr, Rr, rr))
    X = rng.standard_normal((rl, 4, nvec, rr))
    ref = oracle.local_matvec_batched(phiL, A, phiR, X)
    tt.tt_debug_set_fused(mode)
    try:
        tt.tt_trace_enable(64)
        Y = h(tt.tt_local_matvec_batched(g(phiL), g(A), g(phiR), g(X)))
        recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
        tt.tt_trace_disable()
    finally:
        tt.tt_debug_set_fused(0)
    # the fused kernel ran (one mv_s1 record tagged -12) and no separate S2 launch
    assert any(r["stage"] == "mv_s1" and r["tile"] in (-12, -13, -14) for r in recs), recs
    assert not any(r["stage"] == "mv_s2" for r in recs), recs
    for m in range(nvec):
        assert rel(Y[:, :, m, :], ref[:, :, m, :]) <= TOL, (shape, m)
    # and agrees with the three-stage path to rounding
    tt.tt_debug_set_fused(-1)
    try:
        Y3 = h(tt.tt_local_matvec_batched(g(phiL), g(A), g(phiR), g(X)))
    finally:
        tt.tt_debug_set_fused(0)
    assert rel(Y, Y3) <= 1e-13


def test_fused_ineligible_shapes_fall_back(tt):
    """Shapes outside the fused preconditions take the three-stage path even when forced."""
    import oracle
    rng = np.random.default_rng(5)
    for rl, n, rr, Rl, Rr in [(8, 3, 16, 4, 4), (8, 4, 24, 4, 4), (8, 4, 16, 40, 4), (7, 4, 16, 4, 4),
                              (8, 4, 16, 4, 6)]:
        phiL = rng.standard_normal((rl, Rl, rl))
        A = rng.standard_normal((Rl, n, n, Rr))
        phiR = rng.standard_normal((rr, Rr, rr))
        X = rng.standard_normal((rl, n, 2, rr))
        tt.tt_debug_set_fused(1)
        try:
            tt.tt_trace_enable(64)
            Y = h(tt.tt_local_matvec_batched(g(phiL), g(A), g(phiR), g(X)))
            recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
            tt.tt_trace_disable()
        finally:
            tt.tt_debug_set_fused(0)
        assert not any(r["tile"] in (-12, -13) for r in recs)
        assert rel(Y, oracle.local_matvec_batched(phiL, A, phiR, X)) <= TOL


def test_public_fused_mode_halves_workspace_and_matches(tt):
    """tt_set_matvec_mode("fused"): the workspace query drops T1, the call runs the fused kernel
    with that smaller workspace and returns bit-identical results; "three_stage" restores both."""
    rl, rr, Rl, Rr, nvec = 64, 64, 36, 36, 4
    rng = np.random.default_rng(11)
    phiL, A = g(rng.standard_normal((rl, Rl, rl))), g(rng.standard_normal((Rl, 4, 4, Rr)))
    phiR, X = g(rng.standard_normal((rr, Rr, rr))), g(rng.standard_normal((rl, 4, nvec, rr)))
    full = tt.lib.tt_local_matvec_workspace_size(rl, 4, rr, Rl, Rr, nvec)
    Y3 = tt.tt_local_matvec_batched(phiL, A, phiR, X)
    tt.tt_set_matvec_mode("fused")
    try:
        compact = tt.lib.tt_local_matvec_workspace_size(rl, 4, rr, Rl, Rr, nvec)
        t1_bytes = 8 * rl * Rl * 4 * nvec * rr
        assert full - t1_bytes - 4096 <= compact <= full - t1_bytes
        tt.tt_trace_enable(16)
        Yf = tt.tt_local_matvec_batched(phiL, A, phiR, X)
        recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
        tt.tt_trace_disable()
        assert any(r["tile"] == -12 for r in recs)
        # an ineligible core keeps its T1
        assert tt.lib.tt_local_matvec_workspace_size(rl, 3, rr, Rl, Rr, nvec) >= 8 * rl * Rl * 3 * nvec * rr
    finally:
        tt.tt_set_matvec_mode("auto")
    assert tt.lib.tt_local_matvec_workspace_size(rl, 4, rr, Rl, Rr, nvec) == full
    assert torch.equal(Yf, Y3)


def test_fused_mode_rejects_misaligned_operands(tt):
    rl, rr, Rl, Rr, nvec = 8, 16, 4, 4, 1
    base = torch.randn(rl * 4 * nvec * rr + 1, dtype=torch.float64, device="cuda")
    X = base[1:].view(rl, 4, nvec, rr)   # 8-byte aligned only
    phiL = torch.randn(rl, Rl, rl, dtype=torch.float64, device="cuda")
    A = torch.randn(Rl, 4, 4, Rr, dtype=torch.float64, device="cuda")
    phiR = torch.randn(rr, Rr, rr, dtype=torch.float64, device="cuda")
    ref = tt.tt_local_matvec_batched(phiL, A, phiR, X)      # three-stage handles it
    tt.tt_set_matvec_mode("fused")
    try:
        with pytest.raises(tt.TTError) as ei:
            tt.tt_local_matvec_batched(phiL, A, phiR, X)
        assert "16-byte aligned" in str(ei.value)
        # the thread stays usable
        Y = tt.tt_local_matvec_batched(phiL, A, phiR, X.clone())
    finally:
        tt.tt_set_matvec_mode("auto")
    assert float((Y - ref).norm() / ref.norm()) <= 1e-13   # (the misaligned reference ran the generic kernel)

def test_fused_config5_interior_bit_identical(tt):
    """Full-size config-5 interior core (a = b = 256, al = be = 36, K = 32), the launch
    configuration tools/fused_probe.py and bench.py time: the fused evaluation equals the
    three-stage one bit for bit (same k order in every DMMA accumulator), so the oracle parity
    of test_gpu_parity.py::test_config5_w5_sampled carries over."""
    gen = torch.Generator(device="cuda").manual_seed(3)
    r = lambda *s: torch.randn(*s, dtype=torch.float64, device="cuda", generator=gen)
    phiL, A, phiR, X = r(256, 36, 256), r(36, 4, 4, 36), r(256, 36, 256), r(256, 4, 32, 256)
    Y3 = tt.tt_local_matvec_batched(phiL, A, phiR, X)
    tt.tt_set_matvec_mode("fused")
    try:
        Yf = tt.tt_local_matvec_batched(phiL, A, phiR, X)
    finally:
        tt.tt_set_matvec_mode("auto")
    assert torch.equal(Yf, Y3)


def test_fused_sweep_als_matches_three_stage(tt):
    """tt_sweep_als (the W5 launch configuration) at a reduced config-5 shape under both modes."""
    d, nvec = 6, 4
    r = [1, 4, 16, 64, 16, 4, 1]
    R = [1, 4, 36, 36, 36, 4, 1]
    rng = np.random.default_rng(17)
    xs = [g(rng.standard_normal((r[k], 4, r[k + 1]))) for k in range(d)]
    As = [g(rng.standard_normal((R[k], 4, 4, R[k + 1])) / 6) for k in range(d)]
    Xs = [g(rng.standard_normal((r[k], 4, nvec, r[k + 1]))) for k in range(d)]
    out3 = tt.tt_sweep_als(xs, As, Xs)
    tt.tt_set_matvec_mode("fused")
    try:
        outf = tt.tt_sweep_als(xs, As, Xs)
    finally:
        tt.tt_set_matvec_mode("auto")
    for y3, yf in zip(out3[0], outf[0]):
        assert torch.equal(y3, yf)


def _stages(tt, fn):
    tt.tt_trace_enable(64)
    out = fn()
    recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
    tt.tt_trace_disable()
    return out, recs


def test_auto_policy_selects_fused_for_wide_operator_bonds(tt):
    """TT_MATVEC_AUTO (default): eligible cores whose operator bond fills the kernel's 36-row
    blocks (Rl >= 28) run the fused kernel (with the full workspace as the fallback); narrow
    operator bonds keep the three stages."""
    import oracle
    rng = np.random.default_rng(23)
    rl = rr = 64
    for Rl, Rr, nvec, want in [(36, 36, 1, True), (36, 36, 4, True), (36, 36, 40, True),
                               (16, 16, 1, False), (28, 32, 2, True)]:
        phiL = rng.standard_normal((rl, Rl, rl))
        A = rng.standard_normal((Rl, 4, 4, Rr))
        phiR = rng.standard_normal((rr, Rr, rr))
        X = rng.standard_normal((rl, 4, nvec, rr))
        Y, recs = _stages(tt, lambda: tt.tt_local_matvec_batched(g(phiL), g(A), g(phiR), g(X)))
        assert any(r["tile"] == -12 for r in recs) == want, (Rl, Rr, nvec, recs)
        ref = oracle.local_matvec_batched(phiL, A, phiR, X[:, :, :2, :])
        assert rel(h(Y)[:, :, :2, :], ref) <= TOL


@pytest.mark.parametrize("mode", [0, 2])
def test_interface_updates_through_fused_kernel(tt, mode):
    """Left and right interface updates whose first two products run in the
    fused kernel (AUTO policy at Rl = 36, or forced) against the oracle."""
    import oracle
    rng = np.random.default_rng(29)
    for rl, rr, Rl, Rr in [(64, 80, 36, 32), (96, 64, 28, 36)]:
        A = rng.standard_normal((Rl, 4, 4, Rr))
        x = rng.standard_normal((rl, 4, rr))
        pl = rng.standard_normal((rl, Rl, rl))
        pr = rng.standard_normal((rr, Rr, rr))
        tt.tt_debug_set_fused(mode)
        try:
            outL, recL = _stages(tt, lambda: tt.tt_interface_left(g(pl), g(A), g(x)))
            outR, recR = _stages(tt, lambda: tt.tt_interface_right(g(pr), g(A), g(x)))
        finally:
            tt.tt_debug_set_fused(0)
        assert any(r["tile"] == -12 and r["stage"] == "il_s1" for r in recL), recL
        assert any(r["tile"] == -12 and r["stage"] == "ir_s1" for r in recR), recR
        assert rel(h(outL), oracle.interface_left(pl, A, x)) <= TOL
        assert rel(h(outR), oracle.interface_right(pr, A, x)) <= TOL


@pytest.mark.parametrize("mode", ["auto", "fused"])
@pytest.mark.parametrize("shape", [(66, 80, 28, 36, 3), (64, 64, 36, 36, 1), (70, 96, 33, 8, 2)])
def test_fused_kernel_writes_stay_in_bounds(tt, shape, mode):
    """Guard zones (compute-sanitizer is closed on this pool): the output Y and the workspace --
    under "fused" the compact one without T1 -- sit inside larger sentinel-filled buffers; after
    a matvec and both interface updates through the fused kernel the guards are untouched, the
    inputs unchanged and the results equal to the oracle.  Ragged a' groups (66, 70), k-tile
    padding in both phases (Rl = 33: 132 of 144 k-rows; rl = 66: 66 of 80)."""
    import oracle
    rl, rr, Rl, Rr, nvec = shape
    SENT, GUARD, WGUARD = 4321.5, 512, 1 << 16
    rng = np.random.default_rng(sum(shape) + 3)
    pl, A = rng.standard_normal((rl, Rl, rl)), rng.standard_normal((Rl, 4, 4, Rr))
    pr, X = rng.standard_normal((rr, Rr, rr)), rng.standard_normal((rl, 4, nvec, rr))
    ins = [g(pl), g(A), g(pr), g(X)]
    before = [t.clone() for t in ins]

    def guarded(shp):
        n = int(np.prod(shp))
        big = torch.full((2 * GUARD + n,), SENT, dtype=torch.float64, device="cuda")
        return big, big[GUARD:GUARD + n].view(*shp)

    def intact(big, shp):
        n = int(np.prod(shp))
        return bool((big[:GUARD] == SENT).all()) and bool((big[GUARD + n:] == SENT).all())

    tt.tt_set_matvec_mode(mode)
    try:
        need = tt.lib.tt_local_matvec_workspace_size(rl, 4, rr, Rl, Rr, nvec)
        bigW = torch.full((need + WGUARD,), 0xAB, dtype=torch.uint8, device="cuda")
        bigY, Y = guarded((rl, 4, nvec, rr))
        tt.tt_trace_enable(16)
        tt.tt_local_matvec_batched(*ins, Y, workspace=bigW[:need])
        torch.cuda.synchronize()
        recs = [tt.tt_trace_read(i) for i in range(tt.tt_trace_count())]
        tt.tt_trace_disable()
        assert any(r["tile"] == -12 for r in recs)
        assert intact(bigY, Y.shape) and bool((bigW[need:] == 0xAB).all())
        assert rel(h(Y), oracle.local_matvec_batched(pl, A, pr, X)) <= TOL
        # interface updates of the same core
        x = np.ascontiguousarray(X[:, :, 0, :])
        needi = tt.lib.tt_interface_workspace_size(rl, 4, rr, Rl, Rr)
        bigWi = torch.full((needi + WGUARD,), 0xAB, dtype=torch.uint8, device="cuda")
        bigL, outL = guarded((rr, Rr, rr))
        bigR, outR = guarded((rl, Rl, rl))
        tt.tt_interface_left(ins[0], ins[1], g(x), outL, workspace=bigWi[:needi])
        tt.tt_interface_right(ins[2], ins[1], g(x), outR, workspace=bigWi[:needi])
        torch.cuda.synchronize()
        assert intact(bigL, outL.shape) and intact(bigR, outR.shape)
        assert bool((bigWi[needi:] == 0xAB).all())
        assert rel(h(outL), oracle.interface_left(pl, A, x)) <= TOL
        assert rel(h(outR), oracle.interface_right(pr, A, x)) <= TOL
    finally:
        tt.tt_set_matvec_mode("auto")
    for a, b in zip(ins, before):
        assert torch.equal(a, b)


def test_round_robin_producer_equals_thread0_producer(tt):
    """The stage GEMMs with the round-robin TMA producer (default on tiles of 8+ warps) and with
    thread 0 as the producer (debug bit 30) run the same arithmetic: bit-identical results on a
    shape that takes the 12-warp 128 x 144 and the 16-warp 128 x 128 tiles (three-stage path),
    and the fused kernel's three producer placements agree bit for bit as well."""
    gen = torch.Generator(device="cuda").manual_seed(5)
    r = lambda *s: torch.randn(*s, dtype=torch.float64, device="cuda", generator=gen)
    phiL, A, phiR, X = r(256, 36, 256), r(36, 4, 4, 36), r(256, 36, 256), r(256, 4, 8, 256)
    outs = {}
    for name, fused, flags in [("rr", -1, 0), ("t0", -1, 1 << 30), ("f_rr", 2, 0), ("f_t0", 98, 0),
                               ("f_pw", 194, 0)]:
        tt.tt_debug_set_fused(fused)
        tt.tt_debug_set_flags(flags)
        try:
            outs[name] = tt.tt_local_matvec_batched(phiL, A, phiR, X)
        finally:
            tt.tt_debug_set_fused(0)
            tt.tt_debug_set_flags(0)
    for name in ("t0", "f_rr", "f_t0", "f_pw"):
        assert torch.equal(outs[name], outs["rr"]), name


def test_auto_falls_back_for_misaligned_operands(tt):
    """TT_MATVEC_AUTO keeps T1 in the workspace: an 8-byte-aligned X (or phiL) on an eligible
    core silently takes the stage GEMMs and still matches the oracle."""
    import oracle
    rl, rr, Rl, Rr, nvec = 64, 64, 36, 36, 2
    rng = np.random.default_rng(41)
    phiL, A = rng.standard_normal((rl, Rl, rl)), rng.standard_normal((Rl, 4, 4, Rr))
    phiR, X = rng.standard_normal((rr, Rr, rr)), rng.standard_normal((rl, 4, nvec, rr))
    base = torch.empty(X.size + 1, dtype=torch.float64, device="cuda")
    Xm = base[1:].view(rl, 4, nvec, rr)
    Xm.copy_(g(X))
    Y, recs = _stages(tt, lambda: tt.tt_local_matvec_batched(g(phiL), g(A), g(phiR), Xm))
    assert not any(r["tile"] == -12 for r in recs)
    assert rel(h(Y), oracle.local_matvec_batched(phiL, A, phiR, X)) <= TOL
    Y2, recs2 = _stages(tt, lambda: tt.tt_local_matvec_batched(g(phiL), g(A), g(phiR), g(X)))
    assert any(r["tile"] == -12 for r in recs2)
    assert rel(h(Y2), h(Y)) <= 1e-13
