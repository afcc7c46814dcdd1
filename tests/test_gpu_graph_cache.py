"""The eager-call graph cache (tt_set_graph_cache, csrc/tt_core.cu graph_cached): from the second
identical call on, a multi-launch call is replayed from a captured CUDA graph.  Replays must
give exactly the results of the direct path, follow new input VALUES in the same buffers, and
distinguish calls that differ in any pointer or extent."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2509_11890_b200 as m
    return m


def g(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_matvec_replay_matches_direct_and_tracks_values(tt):
    import ttgen
    inp = ttgen.make_inputs(3)
    k = 5
    x, A = g(inp.x[k]), g(inp.A[k])
    rng = np.random.default_rng(7)
    pl = g(rng.standard_normal((x.shape[0], A.shape[0], x.shape[0])))
    pr = g(rng.standard_normal((x.shape[2], A.shape[3], x.shape[2])))
    ws = torch.empty(tt.tt_local_matvec_workspace_size(x.shape[0], x.shape[1], x.shape[2],
                                                       A.shape[0], A.shape[3], 1),
                     dtype=torch.uint8, device="cuda")
    tt.tt_set_graph_cache(False)
    y_direct = tt.tt_local_matvec(pl, A, pr, x, workspace=ws)
    tt.tt_set_graph_cache(True)
    y = torch.empty_like(x)
    outs = []
    for _ in range(4):   # direct, capture + replay, replay, replay
        tt.tt_local_matvec(pl, A, pr, x, y, workspace=ws)
        n = tt.tt_last_launch_count()
        outs.append(y.clone())
        assert n >= 3
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, y_direct)
    # same buffers, new values: the replay reads them
    x.mul_(-2.0)
    tt.tt_local_matvec(pl, A, pr, x, y, workspace=ws)
    torch.cuda.synchronize()
    assert torch.equal(y, -2.0 * y_direct)


def test_sweeps_replay_match_cache_off(tt):
    import ttgen
    inp = ttgen.make_inputs(2)
    x = [g(c) for c in inp.x]
    A = [g(c) for c in inp.A]
    tt.tt_set_graph_cache(False)
    y0, pl0, pr0 = tt.tt_sweep_w34(x, A)
    sl0, sr0 = tt.tt_sweep_interfaces(x, A)
    tt.tt_set_graph_cache(True)
    tr = tt._Train(x, A)
    ws = torch.empty(tt.tt_sweep_w34_workspace_size(tr), dtype=torch.uint8, device="cuda")
    pl, pr = tt.alloc_interfaces(x, A), tt.alloc_interfaces(x, A)
    y = [torch.empty_like(c) for c in x]
    for _ in range(3):
        for t in y + pl + pr:
            t.fill_(float("nan"))
        tt.tt_sweep_w34(x, A, pl, pr, y, workspace=ws)
        torch.cuda.synchronize()
        for a, b in zip(y + pl + pr, y0 + pl0 + pr0):
            assert torch.equal(a, b)
    ql, qr = tt.alloc_interfaces(x, A), tt.alloc_interfaces(x, A)
    for _ in range(3):
        tt.tt_sweep_interfaces(x, A, ql, qr)
        torch.cuda.synchronize()
        for a, b in zip(ql + qr, sl0 + sr0):
            assert torch.equal(a, b)
    # a different output buffer is a different key (no stale replay into the old buffer)
    y2 = [torch.empty_like(c) for c in x]
    tt.tt_sweep_w34(x, A, pl, pr, y2, workspace=ws)
    torch.cuda.synchronize()
    for a, b in zip(y2, y0):
        assert torch.equal(a, b)


def test_interface_replay_and_user_capture(tt):
    import ttgen
    inp = ttgen.make_inputs(3)
    k = 4
    x, A = g(inp.x[k]), g(inp.A[k])
    rng = np.random.default_rng(3)
    phi = g(rng.standard_normal((x.shape[0], A.shape[0], x.shape[0])))
    ref = tt.tt_interface_left(phi, A, x)
    out = torch.empty_like(ref)
    for _ in range(3):
        tt.tt_interface_left(phi, A, x, out)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    # inside the user's own capture the cache is bypassed (the kernels land in the user graph)
    s = torch.cuda.Stream()
    out2 = torch.zeros_like(ref)
    ws = torch.empty(tt.tt_interface_workspace_size(x.shape[0], x.shape[1], x.shape[2], A.shape[0],
                                                    A.shape[3]), dtype=torch.uint8, device="cuda")
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            tt.tt_interface_left(phi, A, x, out2, workspace=ws, stream=s)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out2, ref)


def test_prepared_calls_reissue_the_same_work(tt):
    """tt.prepare: one validation / marshalling, then re-issues of the identical C-ABI call
    (its internally allocated workspace stays alive)."""
    import gc
    import ttgen
    inp = ttgen.make_inputs(3)
    x = [g(c) for c in inp.x]
    A = [g(c) for c in inp.A]
    y0, pl0, pr0 = tt.tt_sweep_w34(x, A)
    p = tt.prepare(tt.tt_sweep_w34, x, A)
    gc.collect()
    torch.cuda.empty_cache()
    for _ in range(3):
        y, pl, pr = p()
        torch.cuda.synchronize()
        for a, b in zip(y + pl + pr, y0 + pl0 + pr0):
            assert torch.equal(a, b)
    k = 5
    rng = np.random.default_rng(11)
    phL = g(rng.standard_normal((x[k].shape[0], A[k].shape[0], x[k].shape[0])))
    phR = g(rng.standard_normal((x[k].shape[2], A[k].shape[3], x[k].shape[2])))
    pm = tt.prepare(tt.tt_local_matvec, phL, A[k], phR, x[k])
    y1 = pm().clone()
    x[k].mul_(2.0)   # a power of two scales every rounded operation exactly
    y2 = pm()
    torch.cuda.synchronize()
    assert torch.equal(y2, 2.0 * y1)
