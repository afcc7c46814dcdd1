/* tt_hotpath.h — C-ABI of the B200 (sm_100a) FP64 tensor-train hot path.
 *
 * The operations are the matrix-free building blocks of the TT Newton-system solve of
 * arXiv 2509.11890 ("An Inexact Tensor-Train Primal-Dual Interior-Point Method for
 * Semidefinite Programs"); PAPER.md = the paper's LaTeX source, cited by line.
 *
 *   TT vector core   x_k in R^{r_k x n_k x r_{k+1}}, r_1 = r_{d+1} = 1
 *   TT matrix core   A_k in R^{R_k x n_row x n_col x R_{k+1}}
 *                    (output/row index i first, input/column index j second)
 *   Block-TT core    X_k in R^{r_k x n_k x nvec x r_{k+1}}
 *   Interface        Phi in R^{r x R x r}, indices [bra, op, ket]: the interface matrices
 *                    T^{<k}, T^{>k} sandwiching the operator's partial
 *                    product, so that the local matvec is the projected operator
 *                    X_{!=k}^T A X_{!=k} applied to a core.
 *
 * Conventions (all calls):
 *  - Every tensor pointer is DEVICE memory, FP64, C-contiguous in the index order written.
 *    Shape/size arguments are host int64.  `stream` is a cudaStream_t passed as void*
 *    (NULL = legacy default stream).
 *  - Ownership: the caller allocates and owns every buffer, including the workspace.  The
 *    library never allocates device memory, frees, or retains a pointer past the call.
 *  - Inputs are never written.  Outputs must not alias inputs (base-pointer equality is
 *    checked -> TT_ERR_ALIASING).
 *  - Validation is synchronous; on any error nothing is enqueued.  Execution is
 *    asynchronous on `stream` (no device synchronisation inside any call), so calls may be
 *    captured into a CUDA graph.  Launch/configuration failures -> TT_ERR_CUDA; faults
 *    during execution surface at the caller's next synchronisation.
 *  - Thread-safe and reentrant; the only mutable state is a thread-local error message.
 *  - Non-finite inputs are not checked; they propagate.
 *  - Arithmetic is IEEE FP64 (DMMA tensor-core FMA); summation order differs from the
 *    paper's plain definition, so results match it to rounding (~1e-15 relative).
 */
#ifndef TT_HOTPATH_H
#define TT_HOTPATH_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TT_OK = 0,
  TT_ERR_INVALID_ARGUMENT = 1, /* non-positive extent, r_1/r_{d+1} or R_1/R_{d+1} != 1, bad flag */
  TT_ERR_NULL_POINTER = 2,
  TT_ERR_ALIASING = 3,         /* an output base pointer equals an input's or another output's */
  TT_ERR_WORKSPACE = 4,        /* workspace NULL or smaller than the *_workspace_size() value */
  TT_ERR_OVERFLOW = 5,         /* an extent product overflows 2^62 elements */
  TT_ERR_CUDA = 6              /* kernel launch / configuration failure (see message) */
} tt_status;

const char* tt_status_string(tt_status s);
/* Detail for the last non-OK status returned on the calling thread ("" if none). */
const char* tt_last_error_message(void);
/* Library version string. */
const char* tt_version(void);

/* ---------------------------------------------------------------------------------------
 * H1-H3  Local matvec  (master formula (M))
 *   y[a',i,b'] = sum_{a,alpha,j,beta,b} phiL[a',alpha,a] A[alpha,i,j,beta] phiR[b',beta,b] x[a,j,b]
 *   phiL (rl,Rl,rl)  A (Rl,n,n,Rr)  phiR (rr,Rr,rr)  x,y (rl,n,rr)
 * Evaluated as the paper's "three matrix products" on DMMA tensor cores,
 * intermediates in the caller's workspace.
 * ------------------------------------------------------------------------------------- */
size_t tt_local_matvec_workspace_size(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                                      int64_t nvec);
tt_status tt_local_matvec(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                          const double* phiL, const double* A, const double* phiR,
                          const double* x, double* y,
                          void* workspace, size_t workspace_bytes, void* stream);

/* H4  Batched Krylov block: the same map on every column m of a Block-TT core
 *   X, Y (rl, n, nvec, rr)   [PAPER.md:294-300 layout; PAPER.md:488 matrix-free GMRES]
 * Workspace: tt_local_matvec_workspace_size(rl, n, rr, Rl, Rr, nvec). */
tt_status tt_local_matvec_batched(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                                  int64_t nvec, const double* phiL, const double* A,
                                  const double* phiR, const double* X, double* Y,
                                  void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------------
 * H5/H6  Interface updates (one core of the sweep)
 *   left : phiL_next[b',beta,b] = sum x[a',i,b'] phiL_prev[a',alpha,a] A[alpha,i,j,beta] x[a,j,b]
 *          phiL_prev (rl,Rl,rl) -> phiL_next (rr,Rr,rr)
 *   right: phiR_prev[a',alpha,a] = sum x[a',i,b'] A[alpha,i,j,beta] phiR_next[b',beta,b] x[a,j,b]
 *          phiR_next (rr,Rr,rr) -> phiR_prev (rl,Rl,rl)
 * (x is real, so conj(x) = x.)  Workspace: tt_interface_workspace_size(...).
 * ------------------------------------------------------------------------------------- */
size_t tt_interface_workspace_size(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr);
tt_status tt_interface_left(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                            const double* phiL_prev, const double* A, const double* x,
                            double* phiL_next,
                            void* workspace, size_t workspace_bytes, void* stream);
tt_status tt_interface_right(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                             const double* phiR_next, const double* A, const double* x,
                             double* phiR_prev,
                             void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------------
 * H7  Sweep: chain the interface updates over d cores from the boundary values
 *     T^{<1} = T^{>d} = 1.
 *   n[d], r[d+1], R[d+1], x_cores[d], A_cores[d], phiL[d+1], phiR[d+1] are HOST arrays; the
 *   pointers they hold are device pointers.  x_cores[k] (r[k],n[k],r[k+1]),
 *   A_cores[k] (R[k],n[k],n[k],R[k+1]).
 *   phiL[k], k=0..d: interface of cores 0..k-1, shape (r[k],R[k],r[k]); phiL[0] is set to 1.
 *   phiR[k], k=0..d: interface of cores k..d-1, shape (r[k],R[k],r[k]); phiR[d] is set to 1.
 *   The local matvec at core k uses phiL[k] and phiR[k+1]; phiL[d] == phiR[0] == x^T A x.
 *   directions: TT_SWEEP_LEFT, TT_SWEEP_RIGHT or TT_SWEEP_BOTH; a NULL phiL / phiR array
 *   skips that direction.
 * ------------------------------------------------------------------------------------- */
enum { TT_SWEEP_LEFT = 1, TT_SWEEP_RIGHT = 2, TT_SWEEP_BOTH = 3 };
size_t tt_sweep_workspace_size(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R);
tt_status tt_sweep_interfaces(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R,
                              const double* const* x_cores, const double* const* A_cores,
                              double* const* phiL, double* const* phiR, int directions,
                              void* workspace, size_t workspace_bytes, void* stream);

/* H7 with the local matvecs interleaved: the ALS/AMEn sweep skeleton with the cores held
 * fixed (SURVEY.md §8(c) reading R9, workload "W5"):
 *   build phiR[d-1..1] right-to-left; then for k = 0..d-1: Y_fwd[k] = local matvec of
 *   X_blocks[k] (Block-TT, nvec columns) with phiL[k], A_cores[k], phiR[k+1], then
 *   phiL[k+1] if k < d-1; then for k = d-1..0: Y_bwd[k] = local matvec, then phiR[k] if k > 0.
 *   X_blocks[k], Y_fwd[k], Y_bwd[k]: (r[k], n[k], nvec, r[k+1]); Y_bwd may be NULL (the
 *   backward pass then overwrites Y_fwd).  phiL/phiR as in tt_sweep_interfaces (both required).
 * Workspace: tt_sweep_als_workspace_size(d, n, r, R, nvec). */
size_t tt_sweep_als_workspace_size(int64_t d, const int64_t* n, const int64_t* r,
                                   const int64_t* R, int64_t nvec);
tt_status tt_sweep_als(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R,
                       int64_t nvec, const double* const* x_cores,
                       const double* const* A_cores, const double* const* X_blocks,
                       double* const* Y_fwd, double* const* Y_bwd,
                       double* const* phiL, double* const* phiR,
                       void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------------
 * H8  Full unrounded TT-matrix x TT-vector product ("ranks grow"; residuals
 *     A vec_TT(X)):
 *   z_k[(a,alpha), i, (b,beta)] = sum_j A_k[alpha,i,j,beta] x_k[a,j,b],
 *   combined bond index a*R[k] + alpha (vector bond major).
 *   A_cores[k] (R[k], n_row[k], n_col[k], R[k+1]), x_cores[k] (r[k], n_col[k], r[k+1]),
 *   z_cores[k] (r[k]*R[k], n_row[k], r[k+1]*R[k+1]).  n_row != n_col allowed.  No workspace.
 * ------------------------------------------------------------------------------------- */
tt_status tt_operator_apply(int64_t d, const int64_t* n_row, const int64_t* n_col,
                            const int64_t* r, const int64_t* R,
                            const double* const* x_cores, const double* const* A_cores,
                            double* const* z_cores, void* stream);

/* ---------------------------------------------------------------------------------------
 * TT rounding ("TT rounding ... to construct an
 * approximation subject to a specified error tolerance delta"; one of its steps moves the
 * block index between cores): Oseledets' algorithm, right-to-left
 * orthonormalisation then left-to-right truncation with per-core threshold
 * delta / sqrt(d-1) * ||T||_F (optionally capped at max_rank > 0), so that
 * ||T - round(T)||_F <= delta ||T||_F.  The orthonormalisation sweep is Householder QR (one
 * thread-block cluster per core, exact to working precision).  The truncating SVDs go through
 * the core unfolding's Gram matrix (DMMA GEMM + a block-Jacobi eigensolver on all SMs) when
 * delta / sqrt(d-1) >= 1e-7 -- numerically zero directions (Gram eigenvalue <= 1e-14 of the
 * largest) are dropped; that route resolves singular values down to ~1e-8 of the largest,
 * ample for the paper's delta = 1e-4 -- and through Householder QR + a
 * one-sided Jacobi SVD of R^T (no squared-condition floor) for tighter tolerances, delta = 0
 * included.
 * cores_in[k] (r_in[k], n[k], r_in[k+1]) device, not modified; cores_out[k] device buffers of
 * at least the input core's size; r_out[d+1] (host) receives the new ranks.  Ranks <= 512.
 * SYNCHRONOUS: the truncation ranks are data dependent (one host read per core).
 * ------------------------------------------------------------------------------------- */
size_t tt_round_workspace_size(int64_t d, const int64_t* n, const int64_t* r);
tt_status tt_round(int64_t d, const int64_t* n, const int64_t* r_in,
                   const double* const* cores_in, double delta, int64_t max_rank, int64_t* r_out,
                   double* const* cores_out, void* workspace, size_t workspace_bytes,
                   void* stream);

/* tt_round_async: the same rounding with every truncation decision taken on
 * the device -- no host read of a singular value, no synchronisation, graph-capturable.  The
 * cores keep host-known STORAGE ranks r_storage[d+1] (host, written before the call returns:
 * r_in, except that a bond wider than its unfolding's other side shrinks to it) and are
 * zero-padded: cores_out[k] is a contiguous (r_storage[k], n[k], r_storage[k+1]) array whose
 * entries with a bond index >= the effective rank are exactly 0, so the padded train
 * represents the rounded tensor as it stands and can be passed to every other entry point;
 * r_dev[d+1] (DEVICE int64) receives the effective ranks (r_dev[0] = r_dev[d] = 1), equal to
 * tt_round's r_out (same formulas and summation order).  A consumer that wants compact cores
 * reads r_dev when convenient and slices.  The truncation route is chosen as in tt_round
 * (Gram matrix for delta / sqrt(d-1) >= 1e-7; below, delta = 0 included, Householder QR + the
 * cluster Jacobi SVD with the singular values ranked and selected on the device).  Other
 * arguments, workspace (tt_round_workspace_size) and errors as tt_round.  The work is that
 * of an untruncated pass (max-rank GEMMs). */
tt_status tt_round_async(int64_t d, const int64_t* n, const int64_t* r_in,
                         const double* const* cores_in, double delta, int64_t max_rank,
                         int64_t* r_storage, int64_t* r_dev, double* const* cores_out,
                         void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------------
 * projected KKT block system action: several
 * operators sharing one frame W_{!=k} act on a Block-TT core whose block index is the KKT
 * component (Delta X_k, Delta Y_k, Delta T_k):
 *   Y[:, :, row, :] = sum_{terms with this row} coeff * L_op( L_op2( X[:, :, col, :] ) )
 * with L_o the projected operator of operator o (its own interfaces phiL[o] (rl,Rl[o],rl),
 * phiR[o] (rr,Rr[o],rr) and core A[o] (Rl[o],n,n,Rr[o])); op2 = -1 means a single operator,
 * op2 >= 0 a product of two projected operators, e.g. (W^T L_X W)(W^T A_eq^T W).
 *   X, Y (rl, n, nblocks, rr); Rl, Rr, phiL, A, phiR, terms are HOST arrays (pointers in
 *   them are device pointers).  Workspace: tt_block_local_matvec_workspace_size(...).
 * ------------------------------------------------------------------------------------- */
typedef struct {
  int64_t row, col, op, op2;
  double coeff;
} tt_block_term;
size_t tt_block_local_matvec_workspace_size(int64_t rl, int64_t n, int64_t rr, int64_t nops,
                                            const int64_t* Rl, const int64_t* Rr);
tt_status tt_block_local_matvec(int64_t rl, int64_t n, int64_t rr, int64_t nblocks, int64_t nops,
                                const int64_t* Rl, const int64_t* Rr, const double* const* phiL,
                                const double* const* A, const double* const* phiR,
                                int64_t nterms, const tt_block_term* terms, const double* X,
                                double* Y, void* workspace, size_t workspace_bytes,
                                void* stream);

/* ---------------------------------------------------------------------------------------
 * two-site (DMRG supercore) local matvec: the projected operator of a
 * PAIR of neighbouring cores ("operates on pairs of neighbouring cores simultaneously",
 * PAPER.md:556-567) applied to nvec supercores:
 *   Y[a',i1,i2,m,b'] = sum phiL[a',al,a] A1[al,i1,j1,g] A2[g,i2,j2,be] phiR[b',be,b] W[a,j1,j2,m,b]
 *   phiL (rl,Rl,rl), A1 (Rl,n1,n1,Rm), A2 (Rm,n2,n2,Rr), phiR (rr,Rr,rr),
 *   W, Y (rl, n1, n2, nvec, rr) (Block-TT layout of the supercore).
 * Evaluated by merging the two operator cores (a small kernel) and running the single-site
 * batched matvec with mode n1*n2.  Workspace: tt_local_matvec_two_site_workspace_size(...).
 * ------------------------------------------------------------------------------------- */
size_t tt_local_matvec_two_site_workspace_size(int64_t rl, int64_t n1, int64_t n2, int64_t rr,
                                               int64_t Rl, int64_t Rm, int64_t Rr, int64_t nvec);
tt_status tt_local_matvec_two_site(int64_t rl, int64_t n1, int64_t n2, int64_t rr, int64_t Rl,
                                   int64_t Rm, int64_t Rr, int64_t nvec, const double* phiL,
                                   const double* A1, const double* A2, const double* phiR,
                                   const double* W, double* Y, void* workspace,
                                   size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------------
 * matrix-free local solve: restarted GMRES(m), or its accelerated
 * variant LGMRES(m, k_aug) ("we employ the accelerated GMRES method [Baker 2005]":
 * each cycle's search space is augmented with the k_aug most recent cycle corrections), on
 * the projected local operator ("solve them in a matrix-free fashion via GMRES
 * ... perform the constituent multiplications sequentially"), for nvec <= 64 independent
 * right-hand sides:
 *   (X_{!=k}^T A X_{!=k}) y_j = f_j,  F, X in the Block-TT layout (rl, n, nvec, rr).
 * Every Arnoldi step is one batched local matvec (H4); orthogonalisation is classical
 * Gram-Schmidt with one re-orthogonalisation pass; Givens rotations per column.  X holds
 * the initial guess on entry and the iterate after `cycles` restart cycles of m steps on
 * exit; a column whose Givens residual estimate |g_{i+1}| / ||f_j|| drops to <= tol is
 * frozen.  rel_res (device, nvec doubles): final relative residual estimate per column;
 * iters (device, nvec int64): Arnoldi steps taken per column.  Fully asynchronous (a fixed
 * launch sequence; no host synchronisation), graph-capturable.
 * Workspace: tt_local_gmres_workspace_size(...) (basis of m+1 Block-TT vectors + matvec).
 * ------------------------------------------------------------------------------------- */
size_t tt_local_gmres_workspace_size(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                                     int64_t nvec, int64_t m, int64_t k_aug);
tt_status tt_local_gmres(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr, int64_t nvec,
                         int64_t m, int64_t k_aug, int64_t cycles, double tol, const double* phiL,
                         const double* A, const double* phiR, const double* F, double* X,
                         double* rel_res, int64_t* iters, void* workspace,
                         size_t workspace_bytes, void* stream);

/* -------------------------------------------------------------------------------------
 * NEXT row 4: matrix-free block LOBPCG for the step-length local
 * generalised eigenproblem ("we minimise -<E, M E> / <E, dM E> via the
 * local eigenvalue problem max vec(E_k)^T E_{!=k}^T dM E_{!=k} vec(E_k) s.t.
 * vec(E_k)^T E_{!=k}^T M E_{!=k} vec(E_k) = 1 ... it can also be implemented in a
 * matrix-free fashion by using iterative eigenvalue solvers (such as LOBPCG [Knyazev 2001])").
 *
 * Computes the nb LARGEST eigenpairs of the pencil (L_A, L_B), L_A = X_{!=k}^T A X_{!=k}
 * (operator A: phiL_A (rl,RlA,rl), A_A (RlA,n,n,RrA), phiR_A (rr,RrA,rr)), L_B likewise from
 * operator B, which must make L_B symmetric positive definite; L_A must be symmetric.
 * phiL_B = A_B = phiR_B = NULL selects L_B = I (RlB, RrB ignored); otherwise all three are
 * required.  For the two-site (DMRG) eigenproblem pass supercore operators merged by
 * tt_merge_operator_cores and n = n1 n2.
 *   X (device, Block-TT layout (rl, n, nb, rr)): initial block on entry (must be L_B-linearly
 *     independent); the L_B-orthonormal Ritz vectors on exit, column j for lam[j].
 *   lam (device, nb): Ritz values, descending.  res (device, nb): ||L_A x - lam L_B x|| /
 *     (||L_A x|| + |lam| ||L_B x||) per column.  iters (device, 1 int64): iterations done.
 *   step (device, 1 double, may be NULL): min(1, 1 / lam[0]) if lam[0] > 0 else 1 -- the
 *     step length of PAPER.md:561-563 when A = -dM, B = M (reading R12).
 * Stops when max_j res_j <= tol or after maxiter iterations; each iteration is one batched
 * local matvec (H4) per operator on nb columns, the residual block L_B-orthogonalised
 * against X, Gram matrices and an on-device Rayleigh-Ritz step (P kept L_B-orthonormal and
 * L_B-orthogonal to X).  refresh > 0: every `refresh` iterations the carried images L_A X,
 * L_B X, L_A P, L_B P are recomputed by matvecs (recommended 20; 0 = never).
 * Fully asynchronous (device-side convergence flag; no host synchronisation), graph-capturable.
 * Workspace: tt_local_lobpcg_workspace_size(...) (RlB = RrB = 0 for B = I).  nb <= 32.
 * ------------------------------------------------------------------------------------- */
size_t tt_local_lobpcg_workspace_size(int64_t rl, int64_t n, int64_t rr, int64_t RlA, int64_t RrA,
                                      int64_t RlB, int64_t RrB, int64_t nb);
tt_status tt_local_lobpcg(int64_t rl, int64_t n, int64_t rr, int64_t RlA, int64_t RrA,
                          int64_t RlB, int64_t RrB, int64_t nb, int64_t maxiter,
                          int64_t refresh, double tol, const double* phiL_A, const double* A_A, const double* phiR_A,
                          const double* phiL_B, const double* A_B, const double* phiR_B,
                          double* X, double* lam, double* res, int64_t* iters, double* step,
                          void* workspace, size_t workspace_bytes, void* stream);
/* Two-site supercore operator ("operates on pairs of neighbouring cores"):
 * A12[al, (i1 i2), (j1 j2), be] = sum_g A1[al, i1, j1, g] A2[g, i2, j2, be];
 * A1 (Rl,n1,n1,Rm), A2 (Rm,n2,n2,Rr), A12 (Rl, n1 n2, n1 n2, Rr), device.  No workspace. */
tt_status tt_merge_operator_cores(int64_t Rl, int64_t n1, int64_t n2, int64_t Rm, int64_t Rr,
                                  const double* A1, const double* A2, double* A12, void* stream);

/* -------------------------------------------------------------------------------------
 * NEXT row 3: core orthonormalisation and the block-index move.
 *
 * tt_orthonormalise: left- (TT_SWEEP_LEFT: cores 0..d-2 left-orthonormal, sum_{a,i}
 * x[a,i,b] x[a,i,b'] = delta_{bb'}, the norm carried into core d-1) or right-
 * (TT_SWEEP_RIGHT: cores 1..d-1 right-orthonormal, the norm carried into core 0)
 * orthonormalisation of a TT vector, the represented tensor unchanged.  Every unfolding is
 * factorised by Householder QR in one thread-block cluster (orthonormal to working precision;
 * a bond wider than the unfolding's other side shrinks to it, r_out); the call is then
 * ASYNCHRONOUS and graph-capturable (r_out is host-known).  An unfolding too large for one
 * cluster's shared memory goes through its Gram matrix and eigendecomposition instead (as
 * tt_round: orthonormal to ~eps kappa^2, exactly rank-deficient bonds shrink); that route
 * reads the ranks on the host, so the call returns synchronised (and cannot be captured).
 * Arguments and workspace as tt_round.
 *
 * tt_block_move_right / _left: "move the block index l to W_{k+1} or W_{k-1} ... by realising
 * one step of the TT rounding procedure".  Right: Wk_hat (r0,n0,l,r1) and
 * Wk1 (r1,n1,r2) -> Wk_out (r0,n0,s) left-orthonormal and Wk1_hat_out (s,n1,l,r2), from the
 * SVD of the (r0 n0) x (l r1) unfolding truncated to the smallest s with
 * ||sigma_{s:}||_2 <= delta ||sigma||_2 (s <= max_rank if max_rank > 0; numerical zeros
 * dropped), so the block tensors W_l are reproduced to relative Frobenius error <= delta.
 * Left: Wkm1 (r0,n0,r1) and Wk_hat (r1,n1,l,r2) -> Wkm1_hat_out (r0,n0,l,s) and Wk_out
 * (s,n1,r2) right-orthonormal, from the (r1 l) x (n1 r2) unfolding.  Outputs are written
 * with the returned extent s (*s_out, host); the caller sizes them for s = min of the
 * unfolding's sides.  The smaller side must be <= 2048.  Synchronous (data-dependent s).
 * Workspace: tt_block_move_workspace_size(r0, n0, l, r1, n1, r2) for the right move with
 * those extents; for the left move pass (r0, n0, l, r1, n1, r2) of its own arguments. *
 * tt_block_move_right_async / _left_async: the same moves with the truncation decided on the
 * device (no host read, no synchronisation, graph-capturable -- a half-sweep of block moves
 * can be one CUDA graph).  The outputs keep the host-known STORAGE extent
 * *s_storage = min of the unfolding's sides and are zero-padded: entries with the new bond
 * index >= the effective rank are exactly 0 (the padded pair represents the same block
 * tensors); *s_dev (DEVICE int64) receives the effective rank, equal to the synchronous
 * call's *s_out.  The work is that of an untruncated move.
 * ------------------------------------------------------------------------------------- */
size_t tt_orthonormalise_workspace_size(int64_t d, const int64_t* n, const int64_t* r);
tt_status tt_orthonormalise(int64_t d, const int64_t* n, const int64_t* r_in,
                            const double* const* cores_in, int direction, int64_t* r_out,
                            double* const* cores_out, void* workspace, size_t workspace_bytes,
                            void* stream);
size_t tt_block_move_workspace_size(int64_t r0, int64_t n0, int64_t l, int64_t r1, int64_t n1,
                                    int64_t r2);
tt_status tt_block_move_right(int64_t r0, int64_t n0, int64_t l, int64_t r1, int64_t n1,
                              int64_t r2, double delta, int64_t max_rank, const double* Wk_hat,
                              const double* Wk1, double* Wk_out, double* Wk1_hat_out,
                              int64_t* s_out, void* workspace, size_t workspace_bytes,
                              void* stream);
tt_status tt_block_move_left(int64_t r0, int64_t n0, int64_t r1, int64_t n1, int64_t l,
                             int64_t r2, double delta, int64_t max_rank, const double* Wkm1,
                             const double* Wk_hat, double* Wkm1_hat_out, double* Wk_out,
                             int64_t* s_out, void* workspace, size_t workspace_bytes,
                             void* stream);
tt_status tt_block_move_right_async(int64_t r0, int64_t n0, int64_t l, int64_t r1, int64_t n1,
                                    int64_t r2, double delta, int64_t max_rank,
                                    const double* Wk_hat, const double* Wk1, double* Wk_out,
                                    double* Wk1_hat_out, int64_t* s_storage, int64_t* s_dev,
                                    void* workspace, size_t workspace_bytes, void* stream);
tt_status tt_block_move_left_async(int64_t r0, int64_t n0, int64_t r1, int64_t n1, int64_t l,
                                   int64_t r2, double delta, int64_t max_rank, const double* Wkm1,
                                   const double* Wk_hat, double* Wkm1_hat_out, double* Wk_out,
                                   int64_t* s_storage, int64_t* s_dev, void* workspace,
                                   size_t workspace_bytes, void* stream);

/* -------------------------------------------------------------------------------------
 * Petrov-Galerkin local operations: the bra train Z differs from the ket train X (ranks
 * rl_bra / rr_bra vs rl / rr).  Interfaces are [bra, op, ket] as everywhere:
 *   phiL (rl_bra, Rl, rl), phiR (rr_bra, Rr, rr).
 * tt_local_matvec_pg: Y = (Z_{!=k}^T A X_{!=k}) X_k column by column, X (rl, n, nvec, rr),
 *   Y (rl_bra, n, nvec, rr_bra) -- with an identity operator core (Rl = Rr = 1) and the
 *   right-hand side train as ket this is the projected right-hand side X_{!=k}^T vec(B) of
 *   the local system; with Z the approximate residual it is the AMEn residual
 *   core.
 * tt_interface_left_pg:  phiL_next (rr_bra, Rr, rr) = sum z[a',i,b'] phiL_prev[a',al,a]
 *   A[al,i,j,be] x[a,j,b];  x_bra = z (rl_bra, n, rr_bra), x_ket = x (rl, n, rr).
 * tt_interface_right_pg: phiR_prev (rl_bra, Rl, rl) = sum z[a',i,b'] A[al,i,j,be]
 *   phiR_next[b',be,b] x[a,j,b].
 * Same conventions as the square calls; one workspace size covers all three.
 * ------------------------------------------------------------------------------------- */
size_t tt_pg_workspace_size(int64_t rl_bra, int64_t rl, int64_t n, int64_t rr_bra, int64_t rr,
                            int64_t Rl, int64_t Rr, int64_t nvec);
tt_status tt_local_matvec_pg(int64_t rl_bra, int64_t rl, int64_t n, int64_t rr_bra, int64_t rr,
                             int64_t Rl, int64_t Rr, int64_t nvec, const double* phiL,
                             const double* A, const double* phiR, const double* X, double* Y,
                             void* workspace, size_t workspace_bytes, void* stream);
tt_status tt_interface_left_pg(int64_t rl_bra, int64_t rl, int64_t n, int64_t rr_bra, int64_t rr,
                               int64_t Rl, int64_t Rr, const double* phiL_prev, const double* A,
                               const double* x_bra, const double* x_ket, double* phiL_next,
                               void* workspace, size_t workspace_bytes, void* stream);
tt_status tt_interface_right_pg(int64_t rl_bra, int64_t rl, int64_t n, int64_t rr_bra, int64_t rr,
                                int64_t Rl, int64_t Rr, const double* phiR_next, const double* A,
                                const double* x_bra, const double* x_ket, double* phiR_prev,
                                void* workspace, size_t workspace_bytes, void* stream);
/* AMEn enrichment (Dolgov & Savostyanov 2014): x_k (rl, n, rx) and the
 * residual core z_k (rl, n, rz) are concatenated along the right bond, x_{k+1} (rx, n1, r2)
 * gets rz zero rows (the represented tensor is unchanged), and the enlarged core is
 * re-orthonormalised by one truncated SVD step (tt_block_move_right with l = 1; delta,
 * max_rank as there): x_k_out (rl, n, s) left-orthonormal, x_k1_out (s, n1, r2), s in *s_out
 * (host), s <= min(rl n, rx + rz).  Synchronous. */
size_t tt_enrich_right_workspace_size(int64_t rl, int64_t n, int64_t rx, int64_t rz, int64_t n1,
                                      int64_t r2);
tt_status tt_enrich_right(int64_t rl, int64_t n, int64_t rx, int64_t rz, int64_t n1, int64_t r2,
                          double delta, int64_t max_rank, const double* x_k, const double* z_k,
                          const double* x_k1, double* x_k_out, double* x_k1_out, int64_t* s_out,
                          void* workspace, size_t workspace_bytes, void* stream);
/* tt_enrich_right_async: the same enrichment with the truncation decided on the device (as
 * tt_block_move_right_async): x_k_out (rl, n, S) and x_k1_out (S, n1, r2) zero-padded to the
 * storage extent *s_storage = S = min(rl n, rx + rz) (host), the effective rank in *s_dev
 * (DEVICE int64).  Asynchronous, graph-capturable. */
tt_status tt_enrich_right_async(int64_t rl, int64_t n, int64_t rx, int64_t rz, int64_t n1,
                                int64_t r2, double delta, int64_t max_rank, const double* x_k,
                                const double* z_k, const double* x_k1, double* x_k_out,
                                double* x_k1_out, int64_t* s_storage, int64_t* s_dev,
                                void* workspace, size_t workspace_bytes, void* stream);

/* Workload W34 as one call: all interfaces (as
 * tt_sweep_interfaces with TT_SWEEP_BOTH: phiL[0..d], phiR[0..d]) and y_k = local matvec of
 * x_k with phiL[k], phiR[k+1] for every core (y_cores[k] shaped like x_cores[k]).  The two
 * chains run concurrently and each matvec starts as soon as its two interfaces exist (event
 * dependencies, pool streams, middle cores first); the caller's stream waits for all of it.
 * The matvec at core k is the same contraction as the left update at core k up to its last
 * stage (phiL[k], A_k and x_k with one vector), so the left chain keeps its stage-2
 * intermediate T2_k (r[k] n[k] R[k+1] r[k+1] doubles per core, in the workspace) and the
 * matvec runs only y_k = T2_k . phiR[k+1] (same results as tt_local_matvec, bit for bit).
 * Asynchronous, graph-capturable.  Workspace: tt_sweep_w34_workspace_size. */
size_t tt_sweep_w34_workspace_size(int64_t d, const int64_t* n, const int64_t* r,
                                   const int64_t* R);
tt_status tt_sweep_w34(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R,
                       const double* const* x_cores, const double* const* A_cores,
                       double* const* phiL, double* const* phiR, double* const* y_cores,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Graph cache for eager calls (default on).  tt_local_matvec(_batched), tt_interface_left/right,
 * tt_sweep_interfaces, tt_sweep_w34 and tt_sweep_als enqueue several kernels per call; the second
 * time a call arrives with the same extents, the same device pointers (host pointer arrays
 * compared by content), the same workspace and the same debug state on the calling thread, it
 * is captured once on an internal stream into a CUDA graph and from then on replayed with one
 * cudaGraphLaunch into the caller's stream (same kernels, same results).  Bypassed while the
 * caller's stream is being captured and while tracing.  Up to 32 graphs per thread (LRU);
 * tt_set_graph_cache(0) disables the cache and destroys its graphs.  A cached graph keeps
 * referring to the device buffers of its key: free or reuse them only as with any pending
 * enqueued work. */
void tt_set_graph_cache(int enabled);

/* Evaluation of the local matvec's three products on the calling thread.
 *   TT_MATVEC_THREE_STAGE: three GEMM launches, both intermediates T1 (a, Rl, n, nvec, b) and
 *     T2 (a, nvec, n, Rr, b) in the workspace.
 *   TT_MATVEC_FUSED: the first two products in one kernel, T1 kept in shared memory tile by
 *     tile (csrc/tt_fused12.cuh): the workspace holds no T1 (about half the bytes) and the
 *     matvec's HBM traffic loses the T1 round trip; same results bit for bit.  Applies to cores
 *     with n = 4, Rl <= 36, Rr <= 36 with Rr % 4 == 0, rr % 16 == 0, rl even and 16-byte aligned
 *     phiL and X; other cores keep the three-stage evaluation and its workspace (a misaligned
 *     phiL / X on an eligible shape returns TT_ERR_INVALID_ARGUMENT in this mode).
 *   TT_MATVEC_AUTO (default): the workspace of TT_MATVEC_THREE_STAGE; the fused kernel on every
 *     eligible core where it was measured faster -- Rl >= 28 and rl, rr >= 64 (the config-5
 *     interior cores: matvecs with any number of columns and every interface update) -- the
 *     three stages elsewhere and whenever phiL / X are not 16-byte aligned.
 * Every *_workspace_size query and every call of the thread (tt_local_matvec(_batched),
 * tt_sweep_als, tt_sweep_w34, tt_block_local_matvec, the local solvers) follows the mode set
 * at the time of the query / call: size the workspace under the mode the call will run in.
 * Returns TT_ERR_INVALID_ARGUMENT for another value. */
typedef enum { TT_MATVEC_AUTO = 0, TT_MATVEC_THREE_STAGE = 1, TT_MATVEC_FUSED = 2 } tt_matvec_mode;
tt_status tt_set_matvec_mode(int mode);

/* Number of kernel launches the last call on this thread enqueued (for a replayed graph: the
 * kernels it contains). */
int64_t tt_last_launch_count(void);

/* ---------------------------------------------------------------------------------------
 * Tracing (measurement support, not part of the math).  While enabled on the calling
 * thread, every kernel the library launches is bracketed by a pair of CUDA events recorded
 * on its own stream, and a record {stage, tile, M, N, K} is appended (M,N,K = GEMM extents;
 * for non-GEMM kernels N = K = 0 and M = elements written).  Do not enable while capturing
 * a CUDA graph.  tt_trace_read synchronises on record i's end event.
 *   stage: TT_ST_PERM, TT_ST_SET, TT_ST_MV_S1..S3 (local matvec), TT_ST_IL_S1..S3 (left
 *   interface), TT_ST_IR_S1..S3 (right interface), TT_ST_APPLY, TT_ST_DAG (one persistent
 *   DAG launch: tile = its task count, M = its tile units).  tile = the GEMM tile's BN.
 * ------------------------------------------------------------------------------------- */
enum {
  TT_ST_PERM = 0, TT_ST_SET = 1,
  TT_ST_MV_S1 = 2, TT_ST_MV_S2 = 3, TT_ST_MV_S3 = 4,
  TT_ST_IL_S1 = 5, TT_ST_IL_S2 = 6, TT_ST_IL_S3 = 7,
  TT_ST_IR_S1 = 8, TT_ST_IR_S2 = 9, TT_ST_IR_S3 = 10,
  TT_ST_APPLY = 11, TT_ST_DAG = 12
};
tt_status tt_trace_enable(int64_t capacity);
tt_status tt_trace_disable(void);
int64_t tt_trace_count(void);
tt_status tt_trace_read(int64_t i, int* stage, int* tile, int64_t* M, int64_t* N, int64_t* K,
                        float* ms);

/* FP64 DMMA throughput probe (roofline denominator): enqueues one kernel of
 * `iters` dependent-free mma.m8n8k4.f64 rounds on every SM; returns its FP64 flop count in
 * *flops.  Time it with events on `stream`. */
tt_status tt_fp64_peak_probe(int64_t iters, double* flops, void* stream);

#ifdef __cplusplus
}
#endif
#include "tt_hotpath_debug.h"   /* test / benchmark hooks (not the production ABI) */
#endif /* TT_HOTPATH_H */
