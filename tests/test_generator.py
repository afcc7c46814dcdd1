"""Input-generator checks (readings R1-R10 of DESIGN.md §3).  CPU only."""
import numpy as np
import pytest

import ttgen
from dense_ref import full_matrix, full_vector, left_interface, unvec_tt_dense, vec_tt_dense


def test_rank_profiles():
    assert ttgen.CONFIGS[1].r == [1, 8, 8, 8, 1] and ttgen.CONFIGS[1].R == [1, 4, 4, 4, 1]
    assert ttgen.CONFIGS[2].r == [1, 4, 16, 32, 32, 32, 16, 4, 1]
    assert ttgen.CONFIGS[2].R == [1] + [9] * 7 + [1]
    assert ttgen.CONFIGS[3].r == [1, 4, 16] + [64] * 5 + [16, 4, 1]
    assert ttgen.CONFIGS[4].r == [1, 4, 16, 64] + [128] * 5 + [64, 16, 4, 1]
    assert ttgen.CONFIGS[4].R == [1, 16] + [25] * 9 + [16, 1]
    assert ttgen.CONFIGS[5].r == [1, 4, 16, 64] + [256] * 5 + [64, 16, 4, 1]
    assert ttgen.CONFIGS[5].R == [1, 16] + [36] * 9 + [16, 1]
    assert ttgen.CONFIGS[5].nvec == 32


def test_deterministic():
    a = ttgen.make_inputs(1)
    b = ttgen.make_inputs(1)
    for u, v in zip(a.x + a.A, b.x + b.A):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("d,rank", [(3, 2), (4, 3)])
def test_kron_sum_spd_and_sylvester(d, rank):
    n = 2
    rng = np.random.default_rng(7)
    X = ttgen.spd_factor(rng, d, n, rank)
    Z = ttgen.spd_factor(rng, d, n, rank)
    Xd, Zd = full_matrix(X), full_matrix(Z)
    assert np.abs(Xd - Xd.T).max() < 1e-13                       # R3 symmetric
    assert np.linalg.eigvalsh(Xd).min() >= d - 1 - 1e-12          # R4 SPD margin
    A = ttgen.kron_sum_operator(X, Z, n)
    Ad = full_matrix(A)
    assert np.abs(Ad - Ad.T).max() < 1e-12
    lam = np.sort(np.linalg.eigvalsh(Ad))
    ref = np.sort((np.linalg.eigvalsh(Xd)[:, None] + np.linalg.eigvalsh(Zd)[None, :]).ravel())
    assert np.abs(lam - ref).max() < 1e-10                        # spectrum {l_i(X)+l_j(Z)}
    M = np.random.default_rng(8).standard_normal((n ** d, n ** d))
    v = vec_tt_dense(M, d, n)
    assert np.allclose(Ad @ v, vec_tt_dense(Xd @ M + M @ Zd.T, d, n), atol=1e-12)
    assert np.array_equal(unvec_tt_dense(v, d, n), M)


def test_config2_structure():
    inp = ttgen.make_inputs(2)
    assert inp.structural_R == [1] + [8] * 7 + [1]
    for k, c in enumerate(inp.A):
        assert c.shape == (inp.cfg.R[k], 4, 4, inp.cfg.R[k + 1])
    # left-orthonormal: Gram of X^{<k} = I
    for k in range(1, inp.cfg.d):
        L = left_interface(inp.x, k)
        assert np.abs(L.T @ L - np.eye(L.shape[1])).max() < 1e-13
    assert abs(np.linalg.norm(full_vector(inp.x)) - 1.0) < 1e-13


def test_config4_structure():
    inp = ttgen.make_inputs(4)
    assert inp.structural_R == [1, 10] + [12] * 9 + [10, 1]   # G rank capped at 4 = N^1 at the ends
    assert inp.X is None


def test_left_right_orthonormalise_preserve_tensor():
    rng = np.random.default_rng(3)
    x = ttgen.gaussian_tt_vector(rng, 4, ttgen.capped_ranks(5, 4, 8))
    v = full_vector(x)
    vl = full_vector(ttgen.left_orthonormalise(x))
    vr = full_vector(ttgen.right_orthonormalise(x))
    assert np.allclose(vl, v / np.linalg.norm(v), atol=1e-13)
    assert np.allclose(vr, v / np.linalg.norm(v), atol=1e-13)
