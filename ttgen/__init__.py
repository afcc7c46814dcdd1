"""Seeded synthetic inputs for the TT hot path — shared by the oracle tests and the CUDA path.

This module is the ONLY code both sides share.  It draws random numbers and assembles TT
cores; it holds none of the hot path's arithmetic (no local matvec, no interface update,
no operator apply).  The recipe is DESIGN.md §3 / SURVEY.md §8(c) readings R1-R10:

* rank profiles (R2): configs 2-5 cap a uniform rank r by the TT-vector bounds
  ``r_k = min(r, N^{k-1}, N^{d+1-k})`` (Def. TT) and the operator rank R by
  ``R_k = min(R, N^{2(k-1)}, N^{2(d+1-k)})``; config 1 uses its explicit lists.
* Gaussian cores (R5): N(0,1) scaled by 1/sqrt(fan-in), fan-in = left bond x input mode.
* Kronecker-sum operators (R1, R3, R4): A = X (x) I + I (x) Z with the core-wise Kronecker
  product of PAPER.md:380-386, X = G_X/||G_X||_F + d*I, G_X core-wise symmetrised, then the
  operator bonds are zero-padded to the configured R.
* left-orthonormalised vectors (R7): Householder QR left-to-right (numpy.linalg.qr).
* RNG (R10): numpy.random.default_rng(seed); draw order = vector cores k=1..d, operator factor
  cores (G_X then G_Z, or A_k), Krylov block k=1..d.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

__all__ = [
    "TTConfig", "CONFIGS", "capped_ranks", "gaussian_tt_vector", "gaussian_tt_matrix",
    "left_orthonormalise", "right_orthonormalise", "kron_sum_operator", "pad_operator",
    "make_inputs", "identity_operator", "random_block",
]


@dataclass
class TTConfig:
    """One BASELINE.json config."""
    index: int
    d: int
    N: int
    r: List[int]
    R: List[int]
    seed: int
    operator: str          # "gaussian" | "kron_sum"
    vector: str            # "gaussian" | "left_qr"
    nvec: int = 1          # Krylov block size (config 5: 32)
    factor_rank: int = 0   # TT rank of G_X, G_Z for kron_sum operators
    workload: str = ""


def capped_ranks(d: int, N: int, r: int) -> List[int]:
    """R2 reading: r_k = min(r, N^{k-1}, N^{d+1-k}), k = 1..d+1 (r_1 = r_{d+1} = 1)."""
    return [int(min(r, N ** (k - 1), N ** (d + 1 - k))) for k in range(1, d + 2)]


def _cfgs() -> List[TTConfig]:
    c1 = TTConfig(1, 4, 4, [1, 8, 8, 8, 1], [1, 4, 4, 4, 1], 0, "gaussian", "gaussian",
                  workload="matvec at all cores + W34 sweep, dense 256x256 check")
    c2 = TTConfig(2, 8, 4, capped_ranks(8, 4, 32), capped_ranks(8, 16, 9), 1, "kron_sum",
                  "left_qr", factor_rank=3, workload="W34 sweep")
    c3 = TTConfig(3, 10, 4, capped_ranks(10, 4, 64), capped_ranks(10, 16, 16), 2, "gaussian",
                  "left_qr", workload="W34 sweep")
    c4 = TTConfig(4, 12, 4, capped_ranks(12, 4, 128), capped_ranks(12, 16, 25), 3, "kron_sum",
                  "gaussian", factor_rank=5, workload="W34 = full sweep at d=12")
    c5 = TTConfig(5, 12, 4, capped_ranks(12, 4, 256), capped_ranks(12, 16, 36), 4, "gaussian",
                  "gaussian", nvec=32, workload="W5 two-direction sweep, batched matvecs K=32")
    return [c1, c2, c3, c4, c5]


CONFIGS = {c.index: c for c in _cfgs()}


def gaussian_tt_vector(rng: np.random.Generator, N: int, r: List[int], scale: bool = True):
    """Cores x_k in R^{r_k x N x r_{k+1}}, N(0,1)/sqrt(r_k N) (R5)."""
    d = len(r) - 1
    cores = []
    for k in range(d):
        c = rng.standard_normal((r[k], N, r[k + 1]))
        if scale:
            c /= np.sqrt(r[k] * N)
        cores.append(c)
    return cores


def gaussian_tt_matrix(rng: np.random.Generator, n_row: int, n_col: int, R: List[int],
                       scale: bool = True):
    """Cores A_k in R^{R_k x n_row x n_col x R_{k+1}}, N(0,1)/sqrt(R_k n_col)."""
    d = len(R) - 1
    cores = []
    for k in range(d):
        c = rng.standard_normal((R[k], n_row, n_col, R[k + 1]))
        if scale:
            c /= np.sqrt(R[k] * n_col)
        cores.append(c)
    return cores


def random_block(rng: np.random.Generator, N: int, r: List[int], nvec: int):
    """Krylov block in the Block-TT layout (r_k, N, nvec, r_{k+1}), R8."""
    d = len(r) - 1
    return [rng.standard_normal((r[k], N, nvec, r[k + 1])) / np.sqrt(r[k] * N) for k in range(d)]


def left_orthonormalise(cores):
    """R7: Householder QR left-to-right on cores 1..d-1, R carried into the next core;
    the last core is normalised to unit Frobenius norm."""
    cores = [c.copy() for c in cores]
    d = len(cores)
    for k in range(d - 1):
        rk, n, rk1 = cores[k].shape
        q, rr = np.linalg.qr(cores[k].reshape(rk * n, rk1))
        if q.shape[1] != rk1:
            raise ValueError("left_orthonormalise needs r_k*n >= r_{k+1} (capped ranks)")
        cores[k] = q.reshape(rk, n, rk1)
        cores[k + 1] = np.tensordot(rr, cores[k + 1], axes=(1, 0))
    cores[-1] = cores[-1] / np.linalg.norm(cores[-1])
    return cores


def right_orthonormalise(cores):
    """R7 mirror: LQ right-to-left on cores d..2; the first core is normalised."""
    cores = [c.copy() for c in cores]
    d = len(cores)
    for k in range(d - 1, 0, -1):
        rk, n, rk1 = cores[k].shape
        q, rr = np.linalg.qr(cores[k].reshape(rk, n * rk1).T)
        if q.shape[1] != rk:
            raise ValueError("right_orthonormalise needs n*r_{k+1} >= r_k (capped ranks)")
        cores[k] = q.T.reshape(rk, n, rk1)
        cores[k - 1] = np.tensordot(cores[k - 1], rr.T, axes=(2, 0))
    cores[0] = cores[0] / np.linalg.norm(cores[0])
    return cores


def identity_operator(d: int, N: int):
    """Rank-1 identity TT matrix (PAPER.md:269 'identity matrix with TT ranks 1', :610)."""
    return [np.eye(N).reshape(1, N, N, 1).copy() for _ in range(d)]


def _tt_matrix_fro_norm(cores) -> float:
    """Frobenius norm of a TT matrix by transfer matrices (input construction only, R4)."""
    e = np.ones((1, 1))
    for c in cores:
        # e'[s', t'] = sum_{s,t,i,j} e[s,t] c[s,i,j,s'] c[t,i,j,t']
        e = np.einsum("st,sijp,tijq->pq", e, c, c)
    return float(np.sqrt(e[0, 0]))


def _tt_sum(a, b):
    """Cores of the TT sum a + b (block structure; ranks add)."""
    d = len(a)
    out = []
    for k in range(d):
        ca, cb = a[k], b[k]
        ra0, n1, n2, ra1 = ca.shape
        rb0, _, _, rb1 = cb.shape
        if d == 1:
            out.append(ca + cb)
        elif k == 0:
            out.append(np.concatenate([ca, cb], axis=3))
        elif k == d - 1:
            out.append(np.concatenate([ca, cb], axis=0))
        else:
            c = np.zeros((ra0 + rb0, n1, n2, ra1 + rb1))
            c[:ra0, :, :, :ra1] = ca
            c[ra0:, :, :, ra1:] = cb
            out.append(c)
    return out


def _kron_cores(a, b):
    """Core-wise Kronecker product of TT matrices, PAPER.md:380-386 (Def. Kronecker product):
    C_k[(s_a,s_b), (i_a,i_b), (j_a,j_b), (t_a,t_b)] = A_k[s_a,i_a,j_a,t_a] B_k[s_b,i_b,j_b,t_b]
    with C-order combined indices."""
    out = []
    for ca, cb in zip(a, b):
        c = np.einsum("aijb,cklg->acikjlbg", ca, cb)
        s = c.shape
        out.append(c.reshape(s[0] * s[1], s[2] * s[3], s[4] * s[5], s[6] * s[7]))
    return out


def spd_factor(rng: np.random.Generator, d: int, n: int, rank: int):
    """R3/R4: X = G/||G||_F + d*I with G a core-wise symmetrised N(0,1) TT matrix of rank
    `rank` (capped); lambda_min(X) >= d - 1 > 0."""
    rg = capped_ranks(d, n * n, rank)
    g = gaussian_tt_matrix(rng, n, n, rg, scale=False)
    g = [(c + c.transpose(0, 2, 1, 3)) / 2.0 for c in g]
    g[0] = g[0] / _tt_matrix_fro_norm(g)
    ident = [np.eye(n).reshape(1, n, n, 1).copy() for _ in range(d)]
    ident[0] = ident[0] * float(d)
    return _tt_sum(g, ident)


def symmetric_tt_matrix(rng: np.random.Generator, d: int, n: int, rank: int, fro: float = 1.0):
    """A symmetric (indefinite) TT matrix of n^d x n^d: core-wise symmetrised N(0,1) cores of
    rank `rank` (capped), scaled to Frobenius norm `fro` (the search direction dX of the
    step-length eigenproblem; reading R12)."""
    rg = capped_ranks(d, n * n, rank)
    g = gaussian_tt_matrix(rng, n, n, rg, scale=False)
    g = [(c + c.transpose(0, 2, 1, 3)) / 2.0 for c in g]
    g[0] = g[0] * (fro / _tt_matrix_fro_norm(g))
    return g


def kron_sum_operator(X, Z, n: int):
    """A = X (x) I + I (x) Z (the L_X-like Kronecker sum of PAPER.md:449), built exactly with
    the core-wise Kronecker product and TT addition; stored rank r_X + r_Z."""
    d = len(X)
    ident = [np.eye(n).reshape(1, n, n, 1).copy() for _ in range(d)]
    return _tt_sum(_kron_cores(X, ident), _kron_cores(ident, Z))


def pad_operator(cores, R: List[int]):
    """Zero-pad the internal operator bonds to the configured ranks R (reading R1)."""
    d = len(cores)
    out = []
    for k, c in enumerate(cores):
        r0, n1, n2, r1 = c.shape
        if r0 > R[k] or r1 > R[k + 1]:
            raise ValueError(f"structural rank ({r0},{r1}) exceeds configured ({R[k]},{R[k+1]})")
        p = np.zeros((R[k], n1, n2, R[k + 1]))
        p[:r0, :, :, :r1] = c
        out.append(p)
    return out


@dataclass
class TTInputs:
    cfg: TTConfig
    x: list                       # vector cores (r_k, N, r_{k+1})
    A: list                       # operator cores (R_k, N, N, R_{k+1})
    X: Optional[list] = None      # Krylov block (r_k, N, nvec, r_{k+1})
    x_right: Optional[list] = None  # right-orthonormalised copy (config 3)
    factors: dict = field(default_factory=dict)  # X_tt, Z_tt for kron_sum configs
    structural_R: Optional[List[int]] = None


def make_inputs(index: int, with_block: Optional[bool] = None) -> TTInputs:
    """Deterministic inputs of BASELINE.json config `index` (1-based), draw order R10."""
    cfg = CONFIGS[index]
    rng = np.random.default_rng(cfg.seed)
    d, N = cfg.d, cfg.N
    x = gaussian_tt_vector(rng, N, cfg.r, scale=(cfg.vector == "gaussian"))
    factors = {}
    structural = None
    if cfg.operator == "gaussian":
        A = gaussian_tt_matrix(rng, N, N, cfg.R)
    else:
        n = int(round(np.sqrt(N)))
        Xf = spd_factor(rng, d, n, cfg.factor_rank)
        Zf = spd_factor(rng, d, n, cfg.factor_rank)
        A0 = kron_sum_operator(Xf, Zf, n)
        structural = [1] + [c.shape[3] for c in A0[:-1]] + [1]
        A = pad_operator(A0, cfg.R)
        factors = {"X": Xf, "Z": Zf}
    x_right = None
    if cfg.vector == "left_qr":
        x_right = right_orthonormalise(x)
        x = left_orthonormalise(x)
    blk = None
    if with_block is None:
        with_block = cfg.nvec > 1
    if with_block:
        blk = random_block(rng, N, cfg.r, cfg.nvec)
    return TTInputs(cfg, x, A, blk, x_right, factors, structural)
