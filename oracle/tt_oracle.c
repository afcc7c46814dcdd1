/* tt_oracle.c — plain, slow, single-threaded CPU ORACLE for the TT hot path (FP64).
 *
 * TEST INFRASTRUCTURE ONLY (see tt_oracle.h).  Nothing here is blocked, fused, vectorised
 * by hand or reordered beyond the paper's own three-product staging (§3.3:
 * "Each matrix-block multiplication with a vector reduces to three matrix products: two
 * with cost O(r^3 R n) and one with cost O(r^2 R^2 n^2)").  Each stage is a plain loop nest
 * over its contraction indices, accumulating in the written index order, with host
 * temporaries.  Index letters (SURVEY.md §8 Notation): a = r_k, b = r_{k+1}, alpha = R_k,
 * beta = R_{k+1}, i = output (row) mode, j = input (column) mode.
 *
 * Build: gcc -O2 -std=c99 -shared -fPIC -o liboracle.so tt_oracle.c   (no -ffast-math)
 */
#include "tt_oracle.h"

#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_INVALID 1
#define OR_NULL 2
#define OR_OVERFLOW 5
#define OR_NOMEM 7

/* product of positive extents with overflow detection (limit 2^62 elements) */
static int mul_ok(int64_t* acc, int64_t v) {
  if (v <= 0) return 0;
  if (*acc > ((int64_t)1 << 62) / v) return 0;
  *acc *= v;
  return 1;
}

static int dims_ok(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr, int64_t* t1,
                   int64_t* t2) {
  int64_t a = 1, b = 1;
  if (rl <= 0 || n <= 0 || rr <= 0 || Rl <= 0 || Rr <= 0) return OR_INVALID;
  /* temporaries T1 (rl,Rl,n,rr) and T2 (rl,n,Rr,rr) — also bound every other extent */
  if (!mul_ok(&a, rl) || !mul_ok(&a, Rl) || !mul_ok(&a, n) || !mul_ok(&a, rr)) return OR_OVERFLOW;
  if (!mul_ok(&b, rl) || !mul_ok(&b, Rr) || !mul_ok(&b, n) || !mul_ok(&b, rr)) return OR_OVERFLOW;
  *t1 = a;
  *t2 = b;
  return OR_OK;
}

/* ---------------------------------------------------------------------------------------
 * Local matvec, master formula (M) of SURVEY.md §8 = X_{!=k}^T A X_{!=k} vec(x_k)
 * (PAPER.md:289-292), as the paper's three matrix products:
 *   S1  T1[a',alpha,j,b] = sum_a          phiL[a',alpha,a] x[a,j,b]
 *   S2  T2[a',i,beta,b]  = sum_{alpha,j}  A[alpha,i,j,beta] T1[a',alpha,j,b]
 *   S3  y[a',i,b']       = sum_{beta,b}   T2[a',i,beta,b] phiR[b',beta,b]
 * ------------------------------------------------------------------------------------- */
int tt_oracle_local_matvec(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                           const double* phiL, const double* A, const double* phiR,
                           const double* x, double* y) {
  int64_t n1, n2, ap, al, a, j, b, i, be, bp;
  double *T1, *T2;
  int st;
  if (!phiL || !A || !phiR || !x || !y) return OR_NULL;
  st = dims_ok(rl, n, rr, Rl, Rr, &n1, &n2);
  if (st) return st;
  T1 = (double*)calloc((size_t)n1, sizeof(double));
  T2 = (double*)calloc((size_t)n2, sizeof(double));
  if (!T1 || !T2) { free(T1); free(T2); return OR_NOMEM; }

  /* S1 */
  for (ap = 0; ap < rl; ++ap)
    for (al = 0; al < Rl; ++al)
      for (a = 0; a < rl; ++a) {
        const double f = phiL[(ap * Rl + al) * rl + a];
        for (j = 0; j < n; ++j)
          for (b = 0; b < rr; ++b)
            T1[((ap * Rl + al) * n + j) * rr + b] += f * x[(a * n + j) * rr + b];
      }
  /* S2 */
  for (ap = 0; ap < rl; ++ap)
    for (al = 0; al < Rl; ++al)
      for (i = 0; i < n; ++i)
        for (j = 0; j < n; ++j)
          for (be = 0; be < Rr; ++be) {
            const double f = A[((al * n + i) * n + j) * Rr + be];
            for (b = 0; b < rr; ++b)
              T2[((ap * n + i) * Rr + be) * rr + b] += f * T1[((ap * Rl + al) * n + j) * rr + b];
          }
  /* S3 */
  for (ap = 0; ap < rl; ++ap)
    for (i = 0; i < n; ++i)
      for (bp = 0; bp < rr; ++bp) {
        double s = 0.0;
        for (be = 0; be < Rr; ++be)
          for (b = 0; b < rr; ++b)
            s += T2[((ap * n + i) * Rr + be) * rr + b] * phiR[(bp * Rr + be) * rr + b];
        y[(ap * n + i) * rr + bp] = s;
      }
  free(T1);
  free(T2);
  return OR_OK;
}

/* (B): the local matvec applied to each column m of a Block-TT core. */
int tt_oracle_local_matvec_batched(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                                   int64_t nvec, const double* phiL, const double* A,
                                   const double* phiR, const double* X, double* Y) {
  int64_t n1, n2, m, a, j, b, len;
  double *xc, *yc;
  int st;
  if (!phiL || !A || !phiR || !X || !Y) return OR_NULL;
  if (nvec <= 0) return OR_INVALID;
  st = dims_ok(rl, n, rr, Rl, Rr, &n1, &n2);
  if (st) return st;
  len = rl * n * rr;
  xc = (double*)malloc((size_t)len * sizeof(double));
  yc = (double*)malloc((size_t)len * sizeof(double));
  if (!xc || !yc) { free(xc); free(yc); return OR_NOMEM; }
  for (m = 0; m < nvec; ++m) {
    for (a = 0; a < rl; ++a)
      for (j = 0; j < n; ++j)
        for (b = 0; b < rr; ++b) xc[(a * n + j) * rr + b] = X[((a * n + j) * nvec + m) * rr + b];
    st = tt_oracle_local_matvec(rl, n, rr, Rl, Rr, phiL, A, phiR, xc, yc);
    if (st) break;
    for (a = 0; a < rl; ++a)
      for (j = 0; j < n; ++j)
        for (b = 0; b < rr; ++b) Y[((a * n + j) * nvec + m) * rr + b] = yc[(a * n + j) * rr + b];
  }
  free(xc);
  free(yc);
  return st;
}

/* ---------------------------------------------------------------------------------------
 * Left interface update (IL): the operator-sandwiched left interface matrix
 * Phi^L_k = (X^{<k+1})^T A^{<k+1} X^{<k+1}, one core at a time:
 *   S1   T1[a',alpha,j,b] = sum_a         phiL[a',alpha,a] x[a,j,b]
 *   S2   T2[a',i,beta,b]  = sum_{alpha,j} A[alpha,i,j,beta] T1[a',alpha,j,b]
 *   S3'  phiL_next[b',beta,b] = sum_{a',i} x[a',i,b'] T2[a',i,beta,b]
 * ------------------------------------------------------------------------------------- */
int tt_oracle_interface_left(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                             const double* phiL_prev, const double* A, const double* x,
                             double* phiL_next) {
  int64_t n1, n2, ap, al, a, j, b, i, be, bp;
  double *T1, *T2;
  int st;
  if (!phiL_prev || !A || !x || !phiL_next) return OR_NULL;
  st = dims_ok(rl, n, rr, Rl, Rr, &n1, &n2);
  if (st) return st;
  T1 = (double*)calloc((size_t)n1, sizeof(double));
  T2 = (double*)calloc((size_t)n2, sizeof(double));
  if (!T1 || !T2) { free(T1); free(T2); return OR_NOMEM; }
  for (ap = 0; ap < rl; ++ap)
    for (al = 0; al < Rl; ++al)
      for (a = 0; a < rl; ++a) {
        const double f = phiL_prev[(ap * Rl + al) * rl + a];
        for (j = 0; j < n; ++j)
          for (b = 0; b < rr; ++b)
            T1[((ap * Rl + al) * n + j) * rr + b] += f * x[(a * n + j) * rr + b];
      }
  for (ap = 0; ap < rl; ++ap)
    for (al = 0; al < Rl; ++al)
      for (i = 0; i < n; ++i)
        for (j = 0; j < n; ++j)
          for (be = 0; be < Rr; ++be) {
            const double f = A[((al * n + i) * n + j) * Rr + be];
            for (b = 0; b < rr; ++b)
              T2[((ap * n + i) * Rr + be) * rr + b] += f * T1[((ap * Rl + al) * n + j) * rr + b];
          }
  for (bp = 0; bp < rr; ++bp)
    for (be = 0; be < Rr; ++be)
      for (b = 0; b < rr; ++b) phiL_next[(bp * Rr + be) * rr + b] = 0.0;
  for (ap = 0; ap < rl; ++ap)
    for (i = 0; i < n; ++i)
      for (bp = 0; bp < rr; ++bp) {
        const double f = x[(ap * n + i) * rr + bp];
        for (be = 0; be < Rr; ++be)
          for (b = 0; b < rr; ++b)
            phiL_next[(bp * Rr + be) * rr + b] += f * T2[((ap * n + i) * Rr + be) * rr + b];
      }
  free(T1);
  free(T2);
  return OR_OK;
}

/* ---------------------------------------------------------------------------------------
 * Right interface update (IR), mirror of (IL) with T^{>k}:
 *   S1''  T1[a,j,b',beta]   = sum_b          x[a,j,b] phiR[b',beta,b]
 *   S2''  T2[a,alpha,i,b']  = sum_{j,beta}   A[alpha,i,j,beta] T1[a,j,b',beta]
 *   S3''  phiR_prev[a',alpha,a] = sum_{i,b'} x[a',i,b'] T2[a,alpha,i,b']
 * ------------------------------------------------------------------------------------- */
int tt_oracle_interface_right(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                              const double* phiR_next, const double* A, const double* x,
                              double* phiR_prev) {
  int64_t n1, n2, ap, al, a, j, b, i, be, bp;
  double *T1, *T2;
  int st;
  if (!phiR_next || !A || !x || !phiR_prev) return OR_NULL;
  st = dims_ok(rl, n, rr, Rl, Rr, &n1, &n2);
  if (st) return st;
  /* T1 (rl,n,rr,Rr) has n*rl*rr*Rr elements; T2 (rl,Rl,n,rr) has n1 elements */
  T1 = (double*)calloc((size_t)n2, sizeof(double));
  T2 = (double*)calloc((size_t)n1, sizeof(double));
  if (!T1 || !T2) { free(T1); free(T2); return OR_NOMEM; }
  for (a = 0; a < rl; ++a)
    for (j = 0; j < n; ++j)
      for (bp = 0; bp < rr; ++bp)
        for (be = 0; be < Rr; ++be) {
          double s = 0.0;
          for (b = 0; b < rr; ++b) s += x[(a * n + j) * rr + b] * phiR_next[(bp * Rr + be) * rr + b];
          T1[((a * n + j) * rr + bp) * Rr + be] = s;
        }
  for (a = 0; a < rl; ++a)
    for (al = 0; al < Rl; ++al)
      for (i = 0; i < n; ++i)
        for (bp = 0; bp < rr; ++bp) {
          double s = 0.0;
          for (j = 0; j < n; ++j)
            for (be = 0; be < Rr; ++be)
              s += A[((al * n + i) * n + j) * Rr + be] * T1[((a * n + j) * rr + bp) * Rr + be];
          T2[((a * Rl + al) * n + i) * rr + bp] = s;
        }
  for (ap = 0; ap < rl; ++ap)
    for (al = 0; al < Rl; ++al)
      for (a = 0; a < rl; ++a) {
        double s = 0.0;
        for (i = 0; i < n; ++i)
          for (bp = 0; bp < rr; ++bp)
            s += x[(ap * n + i) * rr + bp] * T2[((a * Rl + al) * n + i) * rr + bp];
        phiR_prev[(ap * Rl + al) * rl + a] = s;
      }
  free(T1);
  free(T2);
  return OR_OK;
}

/* ---------------------------------------------------------------------------------------
 * Sweep (H7): chain (IL) left-to-right and (IR) right-to-left over the d cores, starting
 * from the boundary values T^{<1} = T^{>d} = 1.
 * ------------------------------------------------------------------------------------- */
int tt_oracle_sweep_interfaces(int64_t d, const int64_t* n, const int64_t* r, const int64_t* R,
                               const double* const* x_cores, const double* const* A_cores,
                               double* const* phiL, double* const* phiR, int directions) {
  int64_t k;
  int st;
  if (d <= 0) return OR_INVALID;
  if (!n || !r || !R || !x_cores || !A_cores) return OR_NULL;
  if (directions < 1 || directions > 3) return OR_INVALID;
  if (r[0] != 1 || r[d] != 1 || R[0] != 1 || R[d] != 1) return OR_INVALID;
  for (k = 0; k < d; ++k) {
    if (n[k] <= 0 || r[k] <= 0 || R[k] <= 0) return OR_INVALID;
    if (!x_cores[k] || !A_cores[k]) return OR_NULL;
  }
  if ((directions & 1) && phiL) {
    for (k = 0; k <= d; ++k)
      if (!phiL[k]) return OR_NULL;
    phiL[0][0] = 1.0;
    for (k = 0; k < d; ++k) {
      st = tt_oracle_interface_left(r[k], n[k], r[k + 1], R[k], R[k + 1], phiL[k], A_cores[k],
                                    x_cores[k], phiL[k + 1]);
      if (st) return st;
    }
  }
  if ((directions & 2) && phiR) {
    for (k = 0; k <= d; ++k)
      if (!phiR[k]) return OR_NULL;
    phiR[d][0] = 1.0;
    for (k = d - 1; k >= 0; --k) {
      st = tt_oracle_interface_right(r[k], n[k], r[k + 1], R[k], R[k + 1], phiR[k + 1],
                                     A_cores[k], x_cores[k], phiR[k]);
      if (st) return st;
    }
  }
  return OR_OK;
}

/* ---------------------------------------------------------------------------------------
 * Unrounded TT-matrix x TT-vector product (AP), PAPER.md:278 (ranks multiply), 440-443:
 *   z_k[(a,alpha), i, (b,beta)] = sum_j A_k[alpha,i,j,beta] x_k[a,j,b]
 * ------------------------------------------------------------------------------------- */
/* One core of (AP): z[(a,alpha), i, (b,beta)] = sum_j A[alpha,i,j,beta] x[a,j,b]. */
int tt_oracle_apply_core(int64_t rl, int64_t ni, int64_t nj, int64_t rr, int64_t Rl, int64_t Rr,
                         const double* x, const double* A, double* z) {
  int64_t a, al, i, j, b, be, t = 1;
  if (!x || !A || !z) return OR_NULL;
  if (rl <= 0 || ni <= 0 || nj <= 0 || rr <= 0 || Rl <= 0 || Rr <= 0) return OR_INVALID;
  if (!mul_ok(&t, rl) || !mul_ok(&t, Rl) || !mul_ok(&t, ni) || !mul_ok(&t, rr) || !mul_ok(&t, Rr))
    return OR_OVERFLOW;
  for (a = 0; a < rl; ++a)
    for (al = 0; al < Rl; ++al)
      for (i = 0; i < ni; ++i)
        for (b = 0; b < rr; ++b)
          for (be = 0; be < Rr; ++be) {
            double s = 0.0;
            for (j = 0; j < nj; ++j)
              s += A[((al * ni + i) * nj + j) * Rr + be] * x[(a * nj + j) * rr + b];
            z[(((a * Rl + al) * ni + i) * rr + b) * Rr + be] = s;
          }
  return OR_OK;
}

int tt_oracle_operator_apply(int64_t d, const int64_t* n_row, const int64_t* n_col,
                             const int64_t* r, const int64_t* R,
                             const double* const* x_cores, const double* const* A_cores,
                             double* const* z_cores) {
  int64_t k;
  int st;
  if (d <= 0) return OR_INVALID;
  if (!n_row || !n_col || !r || !R || !x_cores || !A_cores || !z_cores) return OR_NULL;
  if (r[0] != 1 || r[d] != 1 || R[0] != 1 || R[d] != 1) return OR_INVALID;
  for (k = 0; k < d; ++k) {
    if (n_row[k] <= 0 || n_col[k] <= 0 || r[k] <= 0 || R[k] <= 0) return OR_INVALID;
    if (!x_cores[k] || !A_cores[k] || !z_cores[k]) return OR_NULL;
  }
  for (k = 0; k < d; ++k) {
    st = tt_oracle_apply_core(r[k], n_row[k], n_col[k], r[k + 1], R[k], R[k + 1], x_cores[k],
                              A_cores[k], z_cores[k]);
    if (st) return st;
  }
  return OR_OK;
}

/* ---------------------------------------------------------------------------------------
 * Two-site (DMRG supercore) local matvec, SURVEY.md 8(f) row 4 ("the
 * algorithm operates on pairs of neighbouring cores simultaneously"): the projected operator
 * X_{!=k,k+1}^T A X_{!=k,k+1} applied to a supercore w[a, j1, j2, b], as four products:
 *   S1  T1[a',al,j1,j2,b] = sum_a          phiL[a',al,a] w[a,j1,j2,b]
 *   S2  T2[a',i1,g,j2,b]  = sum_{al,j1}    A1[al,i1,j1,g] T1[a',al,j1,j2,b]
 *   S3  T3[a',i1,i2,be,b] = sum_{g,j2}     A2[g,i2,j2,be] T2[a',i1,g,j2,b]
 *   S4  y[a',i1,i2,b']    = sum_{be,b}     T3[a',i1,i2,be,b] phiR[b',be,b]
 * phiL (rl,Rl,rl), A1 (Rl,n1,n1,Rm), A2 (Rm,n2,n2,Rr), phiR (rr,Rr,rr), w,y (rl,n1,n2,rr).
 * ------------------------------------------------------------------------------------- */
int tt_oracle_local_matvec_two_site(int64_t rl, int64_t n1, int64_t n2, int64_t rr, int64_t Rl,
                                    int64_t Rm, int64_t Rr, const double* phiL, const double* A1,
                                    const double* A2, const double* phiR, const double* w,
                                    double* y) {
  int64_t t = 1, u = 1, v = 1;
  int64_t ap, al, a, j1, j2, b, i1, i2, g, be, bp;
  double *T1, *T2, *T3;
  if (!phiL || !A1 || !A2 || !phiR || !w || !y) return OR_NULL;
  if (rl <= 0 || n1 <= 0 || n2 <= 0 || rr <= 0 || Rl <= 0 || Rm <= 0 || Rr <= 0) return OR_INVALID;
  if (!mul_ok(&t, rl) || !mul_ok(&t, Rl) || !mul_ok(&t, n1) || !mul_ok(&t, n2) || !mul_ok(&t, rr))
    return OR_OVERFLOW;
  if (!mul_ok(&u, rl) || !mul_ok(&u, n1) || !mul_ok(&u, Rm) || !mul_ok(&u, n2) || !mul_ok(&u, rr))
    return OR_OVERFLOW;
  if (!mul_ok(&v, rl) || !mul_ok(&v, n1) || !mul_ok(&v, n2) || !mul_ok(&v, Rr) || !mul_ok(&v, rr))
    return OR_OVERFLOW;
  T1 = (double*)calloc((size_t)t, sizeof(double));
  T2 = (double*)calloc((size_t)u, sizeof(double));
  T3 = (double*)calloc((size_t)v, sizeof(double));
  if (!T1 || !T2 || !T3) { free(T1); free(T2); free(T3); return OR_NOMEM; }
  for (ap = 0; ap < rl; ++ap)
    for (al = 0; al < Rl; ++al)
      for (a = 0; a < rl; ++a) {
        const double f = phiL[(ap * Rl + al) * rl + a];
        for (j1 = 0; j1 < n1; ++j1)
          for (j2 = 0; j2 < n2; ++j2)
            for (b = 0; b < rr; ++b)
              T1[(((ap * Rl + al) * n1 + j1) * n2 + j2) * rr + b] +=
                  f * w[((a * n1 + j1) * n2 + j2) * rr + b];
      }
  for (ap = 0; ap < rl; ++ap)
    for (al = 0; al < Rl; ++al)
      for (i1 = 0; i1 < n1; ++i1)
        for (j1 = 0; j1 < n1; ++j1)
          for (g = 0; g < Rm; ++g) {
            const double f = A1[((al * n1 + i1) * n1 + j1) * Rm + g];
            for (j2 = 0; j2 < n2; ++j2)
              for (b = 0; b < rr; ++b)
                T2[(((ap * n1 + i1) * Rm + g) * n2 + j2) * rr + b] +=
                    f * T1[(((ap * Rl + al) * n1 + j1) * n2 + j2) * rr + b];
          }
  for (ap = 0; ap < rl; ++ap)
    for (i1 = 0; i1 < n1; ++i1)
      for (g = 0; g < Rm; ++g)
        for (i2 = 0; i2 < n2; ++i2)
          for (j2 = 0; j2 < n2; ++j2)
            for (be = 0; be < Rr; ++be) {
              const double f = A2[((g * n2 + i2) * n2 + j2) * Rr + be];
              for (b = 0; b < rr; ++b)
                T3[(((ap * n1 + i1) * n2 + i2) * Rr + be) * rr + b] +=
                    f * T2[(((ap * n1 + i1) * Rm + g) * n2 + j2) * rr + b];
            }
  for (ap = 0; ap < rl; ++ap)
    for (i1 = 0; i1 < n1; ++i1)
      for (i2 = 0; i2 < n2; ++i2)
        for (bp = 0; bp < rr; ++bp) {
          double sum = 0.0;
          for (be = 0; be < Rr; ++be)
            for (b = 0; b < rr; ++b)
              sum += T3[(((ap * n1 + i1) * n2 + i2) * Rr + be) * rr + b] * phiR[(bp * Rr + be) * rr + b];
          y[((ap * n1 + i1) * n2 + i2) * rr + bp] = sum;
        }
  free(T1);
  free(T2);
  free(T3);
  return OR_OK;
}
