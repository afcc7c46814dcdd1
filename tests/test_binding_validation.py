"""The Python binding validates shapes and devices BEFORE any pointer reaches the C-ABI
(the library takes its extents from x / A, so a wrongly shaped interface or output
would be read or written out of bounds).  CPU-only: with CPU tensors a consistent call must
stop at the CUDA-tensor check (TypeError, no CPU fallback) and an inconsistent one earlier,
at the shape check (ValueError)."""
import pytest
import torch

tt = pytest.importorskip("paper_2509_11890_b200")


def z(*shape):
    return torch.zeros(*shape, dtype=torch.float64)


RL, N, RR, AL, BE = 5, 4, 6, 3, 2


def good():
    return z(RL, AL, RL), z(AL, N, N, BE), z(RR, BE, RR), z(RL, N, RR)


def test_local_matvec_consistent_reaches_device_check():
    with pytest.raises(TypeError, match="CUDA"):
        tt.tt_local_matvec(*good())


@pytest.mark.parametrize("which,shape", [
    (0, (RL + 1, AL, RL)), (0, (RL, AL + 1, RL)), (1, (AL, N, N, BE + 1)), (1, (AL, N + 1, N, BE)),
    (2, (RR, BE, RR + 1)), (2, (RR, BE + 1, RR)),
])
def test_local_matvec_bad_shapes(which, shape):
    args = list(good())
    args[which] = z(*shape)
    with pytest.raises(ValueError):
        tt.tt_local_matvec(*args)


def test_local_matvec_bad_output():
    phiL, A, phiR, x = good()
    with pytest.raises(ValueError, match="y"):
        tt.tt_local_matvec(phiL, A, phiR, x, y=z(RL, N, RR + 1))
    X = z(RL, N, 3, RR)
    with pytest.raises(ValueError, match="Y"):
        tt.tt_local_matvec_batched(phiL, A, phiR, X, Y=z(RL, N, 2, RR))


def test_interfaces_bad_shapes():
    phiL, A, phiR, x = good()
    with pytest.raises(ValueError, match="phiL_prev"):
        tt.tt_interface_left(phiR, A, x)
    with pytest.raises(ValueError, match="phiL_next"):
        tt.tt_interface_left(phiL, A, x, out=z(RR, BE, RR + 1))
    with pytest.raises(ValueError, match="phiR_next"):
        tt.tt_interface_right(phiL, A, x)
    with pytest.raises(ValueError, match="phiR_prev"):
        tt.tt_interface_right(phiR, A, x, out=z(RL, AL + 1, RL))
    with pytest.raises(TypeError, match="CUDA"):
        tt.tt_interface_left(phiL, A, x)


def train():
    xs = [z(1, N, 3), z(3, N, 4), z(4, N, 1)]
    As = [z(1, N, N, 2), z(2, N, N, 2), z(2, N, N, 1)]
    return xs, As


def test_train_bond_mismatch():
    xs, As = train()
    xs[1] = z(3, N, 5)
    with pytest.raises(ValueError, match="vector bond"):
        tt.tt_sweep_interfaces(xs, As)
    xs, As = train()
    As[1] = z(2, N, N, 3)
    with pytest.raises(ValueError, match="operator bond"):
        tt.tt_sweep_interfaces(xs, As)
    xs, As = train()
    As[2] = z(2, N + 1, N + 1, 1)
    with pytest.raises(ValueError, match="mode"):
        tt.tt_sweep_w34(xs, As)


def test_sweep_output_shapes():
    xs, As = train()
    pl = tt.alloc_interfaces(xs, As)
    pl[2] = z(4, 2, 5)
    with pytest.raises(ValueError, match=r"phiL\[2\]"):
        tt.tt_sweep_interfaces(xs, As, phiL=pl, directions=tt.TT_SWEEP_LEFT)
    ys = [torch.zeros_like(c) for c in xs]
    ys[0] = z(1, N, 4)
    with pytest.raises(ValueError, match=r"y_cores\[0\]"):
        tt.tt_sweep_w34(xs, As, y_cores=ys)
    Xb = [z(c.shape[0], N, 2, c.shape[2]) for c in xs]
    Yb = [torch.zeros_like(c) for c in Xb]
    Yb[1] = z(3, N, 3, 4)
    with pytest.raises(ValueError, match=r"Y_fwd\[1\]"):
        tt.tt_sweep_als(xs, As, Xb, Y_fwd=Yb)


def test_apply_bad_z():
    xs, As = train()
    zs = [z(c.shape[0] * A.shape[0], N, c.shape[2] * A.shape[3]) for c, A in zip(xs, As)]
    zs[1] = z(6, N, 7)
    with pytest.raises(ValueError, match=r"z_cores\[1\]"):
        tt.tt_operator_apply(xs, As, zs)
    As[0] = z(1, N, N + 1, 2)
    with pytest.raises(ValueError, match="column mode"):
        tt.tt_operator_apply(xs, As)


def test_solver_bad_shapes():
    phiL, A, phiR, _ = good()
    F = z(RL, N, 2, RR)
    with pytest.raises(ValueError, match="phiR"):
        tt.tt_local_gmres(phiL, A, phiL, F)
    with pytest.raises(ValueError, match="rel_res"):
        tt.tt_local_gmres(phiL, A, phiR, F, rel_res=z(3))
    with pytest.raises(ValueError, match="lam"):
        tt.tt_local_lobpcg((phiL, A, phiR), z(RL, N, 2, RR), lam=z(3))
    with pytest.raises(ValueError, match="operator 1"):
        tt.tt_block_local_matvec([(phiL, A, phiR), (phiL, A, phiL)], [(0, 0, 0, -1, 1.0)],
                                 z(RL, N, 1, RR))
    with pytest.raises(ValueError, match="indexes outside"):
        tt.tt_block_local_matvec([(phiL, A, phiR)], [(0, 1, 0, -1, 1.0)], z(RL, N, 1, RR))
    with pytest.raises(ValueError, match="x_k1"):
        tt.tt_enrich_right(z(RL, N, 3), z(RL, N, 2), z(4, N, 2))
    with pytest.raises(ValueError):
        tt.tt_block_move_right(z(RL, N, 2, 3), z(4, N, 2))
