/* tt_oracle.h — plain, slow, single-threaded CPU ORACLE for the TT hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code, header,
 * helper or constant with the CUDA path (paper_2509_11890_b200/csrc, include/tt_hotpath.h).
 *
 * Every function takes HOST pointers, FP64, C-contiguous arrays in the index order written
 * (SURVEY.md §8 Notation).  Same argument order as the GPU C-ABI, minus workspace/stream.
 * Return value: 0 = OK, 1 = invalid argument, 2 = NULL pointer, 5 = size overflow,
 * 7 = host allocation failure.
 *
 * Definitions followed (PAPER.md = arXiv 2509.11890 LaTeX source):
 *   local matvec  y = (X_{!=k}^T A X_{!=k}) vec(x_k)            PAPER.md:289-292 (§2.3, ALS)
 *                 evaluated as "three matrix products"           PAPER.md:526 (§3.3)
 *   interfaces    Phi built from interface matrices T^{<k},T^{>k} PAPER.md:244-253 (Def. Interface)
 *   TT matrix     A_k in R^{R_k x n_row x n_col x R_{k+1}}        PAPER.md:270-276 (Def. TT Matrix)
 *   block TT      X_k in R^{r_k x n x nvec x r_{k+1}}             PAPER.md:294-300 (Def. Block TT)
 *   apply         unrounded A x, ranks multiply
 */
#ifndef TT_ORACLE_H
#define TT_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* y[a',i,b'] = sum_{a,alpha,j,beta,b} phiL[a',alpha,a] A[alpha,i,j,beta] phiR[b',beta,b] x[a,j,b]
 * phiL (rl,Rl,rl), A (Rl,n,n,Rr), phiR (rr,Rr,rr), x,y (rl,n,rr). */
int tt_oracle_local_matvec(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                           const double* phiL, const double* A, const double* phiR,
                           const double* x, double* y);

/* The same map applied to every column m of a Block-TT core: X,Y (rl,n,nvec,rr). */
int tt_oracle_local_matvec_batched(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                                   int64_t nvec, const double* phiL, const double* A,
                                   const double* phiR, const double* X, double* Y);

/* phiL_next[b',beta,b] = sum x[a',i,b'] phiL_prev[a',alpha,a] A[alpha,i,j,beta] x[a,j,b] */
int tt_oracle_interface_left(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                             const double* phiL_prev, const double* A, const double* x,
                             double* phiL_next);

/* phiR_prev[a',alpha,a] = sum x[a',i,b'] A[alpha,i,j,beta] phiR_next[b',beta,b] x[a,j,b] */
int tt_oracle_interface_right(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                              const double* phiR_next, const double* A, const double* x,
                              double* phiR_prev);

/* phiL[k] (k=0..d) interface of cores 0..k-1, shape (r[k],R[k],r[k]); phiL[0] := 1.
 * phiR[k] (k=0..d) interface of cores k..d-1, shape (r[k],R[k],r[k]); phiR[d] := 1.
 * directions: 1 = left chain, 2 = right chain, 3 = both.  NULL array skips a direction. */
int tt_oracle_sweep_interfaces(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R,
                               const double* const* x_cores, const double* const* A_cores,
                               double* const* phiL, double* const* phiR, int directions);

/* z_k[(a,alpha), i, (b,beta)] = sum_j A_k[alpha,i,j,beta] x_k[a,j,b], combined a*R[k]+alpha.
 * z_k shape (r[k]*R[k], n_row[k], r[k+1]*R[k+1]). */
int tt_oracle_operator_apply(int64_t d, const int64_t* n_row, const int64_t* n_col,
                             const int64_t* r, const int64_t* R,
                             const double* const* x_cores, const double* const* A_cores,
                             double* const* z_cores);

/* One core of the product above: x (rl,nj,rr), A (Rl,ni,nj,Rr) -> z (rl*Rl, ni, rr*Rr).
 * No boundary-rank condition, so a slice x[a0:a1] gives the matching rows of z_k. */
int tt_oracle_apply_core(int64_t rl, int64_t ni, int64_t nj, int64_t rr, int64_t Rl, int64_t Rr,
                         const double* x, const double* A, double* z);

/* Two-site (DMRG supercore) local matvec:
 * y[a',i1,i2,b'] = sum phiL[a',al,a] A1[al,i1,j1,g] A2[g,i2,j2,be] phiR[b',be,b] w[a,j1,j2,b]
 * phiL (rl,Rl,rl), A1 (Rl,n1,n1,Rm), A2 (Rm,n2,n2,Rr), phiR (rr,Rr,rr), w,y (rl,n1,n2,rr). */
int tt_oracle_local_matvec_two_site(int64_t rl, int64_t n1, int64_t n2, int64_t rr, int64_t Rl,
                                    int64_t Rm, int64_t Rr, const double* phiL, const double* A1,
                                    const double* A2, const double* phiR, const double* w,
                                    double* y);

#ifdef __cplusplus
}
#endif
#endif
