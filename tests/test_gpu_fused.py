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


@pytest.mark.parametrize("mode", [1, 2, 3, 5])
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
    assert any(r["stage"] == "mv_s1" and r["tile"] == -12 for r in recs), recs
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
        assert not any(r["tile"] == -12 for r in recs)
        assert rel(Y, oracle.local_matvec_batched(phiL, A, phiR, X)) <= TOL
