// tt_solvers.cu — the NEXT rows of SURVEY.md §8(f): TT rounding / block moves / enrichment,
// KKT block action, two-site matvec, local GMRES, Petrov-Galerkin operations, LOBPCG.
#include "tt_internal.cuh"
#include <cooperative_groups.h>

namespace ttint {

#include "tt_gmres.cuh"
#include "tt_round.cuh"
#include "tt_qr.cuh"
#include "tt_lobpcg.cuh"

// Symmetric eigendecomposition of the n x n Gram matrix G: lam (descending) and V (columns)
// in the caller's buffers.  n < 24: element-wise cooperative Jacobi (4 padded np x np
// buffers, np = n rounded up to even); larger n: block Jacobi (G and V padded to a multiple
// of 32 -- 64 for the BS = 32 probe variant -- plus the per-pair rotations).  Scratch:
// sym_eigen_scratch(n) doubles.
constexpr int kBlockJacobiMin = 24;   // below: the element-wise kernel (measured faster)
constexpr int kJBig = 64;             // padding granularity of the block kernels (2 BS, BS = 32)
long long sym_eigen_scratch(long long n) {
  const long long np = (n + 1) & ~1LL;
  const long long nb = (n + kJBig - 1) / kJBig * kJBig;
  const long long elem = 4 * np * np, blk = 2 * nb * nb + nb * kJBig;
  return std::max(elem, blk) + 2 * 4096 + 8;
}
thread_local int g_eigen_elementwise = 0;   // test hook: force the element-wise kernel
template <int BS>
static cudaError_t launch_block2(double* G0, double* V0, int np, double* Rbuf, double* part,
                                 cudaStream_t s) {
  using C = Jb2<BS>;
  int per_sm = 0;
  if (cudaError_t e = smem_attr((const void*)jacobi_block2_kernel<BS>, (int)C::kSmem)) return e;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_block2_kernel<BS>, C::kLaunch,
                                                C::kSmem);
  const int m = np / C::B2;
  int grid = num_sms() * std::max(per_sm, 1);
  const int tasks = 2 * m * m;
  if (grid > tasks) grid = tasks;
  int sweeps = 40;
  void* args[] = {&G0, &V0, (void*)&np, &sweeps, &Rbuf, &part};
  return cudaLaunchCooperativeKernel((const void*)jacobi_block2_kernel<BS>, grid, C::kLaunch,
                                     args, C::kSmem, s);
}
cudaError_t launch_sym_eigen(const double* G, double* V, double* lam, int n, double* scratch,
                             cudaStream_t s) {
  g_stage = TT_ST_PERM;
  const long long tr = trace_begin(0, (long long)n * n, 0, 0, s);
  int dev = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaError_t e;
  if (n >= kBlockJacobiMin && !g_eigen_elementwise) {
    // debug bit 16: the first block kernel (BS = 16, full inner sweeps, scalar updates);
    // bit 2: the second kernel with BS = 32 instead of 16 (measured slower below n = 1024)
    const bool v1 = (g_dbg_flags & (1 << 16)) != 0, bs16 = v1 || (g_dbg_flags & (1 << 2)) == 0;
    const int gran = bs16 ? kJB2 : kJBig;
    const int np = (n + gran - 1) / gran * gran;
    const long long NN = (long long)np * np;
    double* G0 = scratch;
    double* V0 = G0 + NN;
    double* Rbuf = V0 + NN;
    const int m = np / gran;   // block pairs per step
    double* part = Rbuf + (long long)m * gran * gran;
    int* which = reinterpret_cast<int*>(part + 2 * 4096);
    long long eb = std::min<long long>(4096, (NN + 255) / 256);
    embed_kernel<<<(unsigned)eb, 256, 0, s>>>(G, G0, n, np);
    ++g_launches;
    if ((e = cudaMemsetAsync(which, 0, sizeof(int), s)) != cudaSuccess) return e;
    if (v1) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_block_coop_kernel, 256, 0);
      int grid = num_sms() * std::max(per_sm, 1);
      const int tasks = m * m + (np / kJB2) * m;
      if (grid > tasks) grid = tasks;
      if (grid > 4096) grid = 4096;
      int sweeps = 40;
      int npi = np;
      void* args[] = {&G0, &V0, (void*)&npi, &sweeps, &Rbuf, &part};
      e = cudaLaunchCooperativeKernel((const void*)jacobi_block_coop_kernel, grid, 256, args, 0, s);
    } else {
      e = bs16 ? launch_block2<16>(G0, V0, np, Rbuf, part, s)
               : launch_block2<32>(G0, V0, np, Rbuf, part, s);
    }
    ++g_launches;
    if (e != cudaSuccess) return e;
    sort_padded_kernel<<<(n + 255) / 256, 256, 0, s>>>(G0, G0, V0, V0, which, V, lam, n, np);
    ++g_launches;
    trace_end(tr, s);
    return cudaGetLastError();
  }
  const int np = (n + 1) & ~1;
  const long long NN = (long long)np * np;
  double* G0 = scratch;
  double* G1 = G0 + NN;
  double* V0 = G1 + NN;
  double* V1 = V0 + NN;
  double* part = V1 + NN;
  int* which = reinterpret_cast<int*>(part + 2 * 4096);
  long long eb = (NN + 255) / 256;
  if (eb > 4096) eb = 4096;
  embed_kernel<<<(unsigned)eb, 256, 0, s>>>(G, G0, n, np);
  ++g_launches;
  const size_t smem = (size_t)np / 2 * (2 * sizeof(double) + 2 * sizeof(int));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_coop_kernel, 256, smem);
  int grid = num_sms() * std::max(per_sm, 1);
  const long long want = std::max<long long>(1, ((long long)(np / 2) * (np / 2) + 255) / 256);
  if (grid > want) grid = (int)want;
  if (grid > 4096) grid = 4096;
  int sweeps = 25;
  void* args[] = {&G0, &G1, &V0, &V1, (void*)&np, &sweeps, &part, &which};
  e = cudaLaunchCooperativeKernel((const void*)jacobi_coop_kernel, grid, 256, args, smem, s);
  ++g_launches;
  if (e != cudaSuccess) return e;
  sort_padded_kernel<<<(n + 255) / 256, 256, 0, s>>>(G0, G1, V0, V1, which, V, lam, n, np);
  ++g_launches;
  trace_end(tr, s);
  return cudaGetLastError();
}

// Block-TT column gather / scaled scatter-add: column `col` of X (rows, nb, rr) <-> v (rows, rr)
__global__ void gather_col_kernel(const double* __restrict__ X, double* __restrict__ v,
                                  long long rows, int nb, int rr, int col) {
  const long long tot = rows * rr;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const long long row = e / rr, b = e - row * rr;
    v[e] = X[(row * nb + col) * rr + b];
  }
}
__global__ void scatter_add_col_kernel(const double* __restrict__ v, double* __restrict__ Y,
                                       long long rows, int nb, int rr, int row_blk, double c) {
  const long long tot = rows * rr;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const long long row = e / rr, b = e - row * rr;
    double* y = Y + (row * nb + row_blk) * rr + b;
    *y = fma(c, v[e], *y);
  }
}

// W[r, c] = V[r * ldv + c] * f[c], r < rows, c < s
__global__ void scale_cols_ld_kernel(const double* __restrict__ V, long long ldv,
                                     const double* __restrict__ f, double* __restrict__ W,
                                     long long rows, int s) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < rows * s;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / s;
    const int c = (int)(e - r * s);
    W[e] = V[r * ldv + c] * f[c];
  }
}

// out (cols x rows) = in (rows x cols)^T, both row-major
__global__ void transpose2d_kernel(const double* __restrict__ in, double* __restrict__ out,
                                   long long rows, long long cols) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < rows * cols;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / cols, j = e - i * cols;
    out[j * rows + i] = in[e];
  }
}
// out (a, l, i, b) = in (a, i, l, b)   (the block index moved next to the left bond)
__global__ void swap_mid_kernel(const double* __restrict__ in, double* __restrict__ out,
                                long long a, long long ni, long long nl, long long b) {
  const long long total = a * ni * nl * b;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    long long r = e;
    const long long bb = r % b; r /= b;
    const long long l = r % nl; r /= nl;
    const long long i = r % ni;
    const long long aa = r / ni;
    out[((aa * nl + l) * ni + i) * b + bb] = in[e];
  }
}

// Two-site supercore operator: A12[al, (i1 i2), (j1 j2), be] = sum_g A1[al,i1,j1,g] A2[g,i2,j2,be]
// (the local operator of a pair of cores; tiny, one thread per output)
__global__ void merge_cores_kernel(const double* __restrict__ A1, const double* __restrict__ A2,
                                   double* __restrict__ A12, long long Rl, long long n1,
                                   long long n2, long long Rm, long long Rr) {
  const long long total = Rl * n1 * n2 * n1 * n2 * Rr;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    long long r = e;
    const long long be = r % Rr; r /= Rr;
    const long long j2 = r % n2; r /= n2;
    const long long j1 = r % n1; r /= n1;
    const long long i2 = r % n2; r /= n2;
    const long long i1 = r % n1;
    const long long al = r / n1;
    double s = 0.0;
    for (long long g = 0; g < Rm; ++g)
      s = fma(A1[((al * n1 + i1) * n1 + j1) * Rm + g], A2[((g * n2 + i2) * n2 + j2) * Rr + be], s);
    A12[e] = s;
  }
}

}  // namespace ttint

using namespace ttint;

extern "C" {

// ---- TT rounding ------------------------------------------------------
size_t tt_round_workspace_size(int64_t d, const int64_t* n, const int64_t* r) {
  if (d <= 0 || !n || !r) return 0;
  long long core_max = 0, rmax = 0, tot = 0;
  bool ok = true;
  for (int64_t k = 0; k < d; ++k) {
    const long long sz = prod({r[k], n[k], r[k + 1]}, ok);
    core_max = std::max(core_max, sz);
    tot += align_up((size_t)sz * 8, 256) / 8 + 32;
  }
  for (int64_t k = 0; k <= d; ++k) rmax = std::max<long long>(rmax, r[k]);
  if (!ok) return 0;
  // working cores, one temp core, G, V, Bm (rmax^2 each), d, lam (rmax), eigen scratch
  return ws_bytes({tot, core_max, rmax * rmax, rmax * rmax, rmax * rmax, rmax, rmax,
                   sym_eigen_scratch(rmax)});
}

// phases: bit 0 = right-to-left orthonormalisation, bit 1 = left-to-right truncation
// (delta = 0, max_rank = 0: plain left-to-right orthonormalisation)
// the selected singular triplets of the accurate truncation (cluster Jacobi SVD of R):
// Usel[r][i] = BJ[r][perm[i]] / sigma[perm[i]] (kk x sk), SJt[i][col] = sigma[perm[i]] J[col][perm[i]]
__global__ void svd_select_kernel(const double* __restrict__ BJ, const double* __restrict__ J,
                                  const int* __restrict__ perm, int kk, int rk1, int sk,
                                  double* __restrict__ Usel, double* __restrict__ SJt) {
  // R^T J = BJ (columns U_R sigma) => R = J BJ^T: left vectors J, sigma-scaled right vectors BJ
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < kk * sk) {
    const int r = e / sk, i = e - r * sk;
    Usel[e] = J[(long long)r * kk + perm[i]];
  }
  if (e < sk * rk1) {
    const int i = e / rk1, col = e - i * rk1;
    SJt[e] = BJ[(long long)col * kk + perm[i]];
  }
}

// Device-side truncation decision of the asynchronous rounding (tt_round_async): from the
// descending Gram eigenvalues lam[0..m) it drops the numerical zeros (lam <= zero_rel lam_0),
// then -- with use_thr -- the longest tail whose Frobenius norm sqrt(sum lam) stays <= thr
// (first core: thr = fac * sqrt(sum lam) is computed here and kept in thr_dev for the later
// cores), caps at max_rank, writes the rank to *r_dev and the two zero-padded m x m factors
// Bm1 = V[:, :sk] diag(lam^-1/2), Bm2 = V[:, :sk] diag(lam^1/2) (columns >= sk exactly zero).
// Same formulas, summation order and IEEE operations as the host loop of tt_round.
__global__ void __launch_bounds__(256) trunc_decide_kernel(
    const double* __restrict__ lam, const double* __restrict__ V, int m, int use_thr, int first,
    double fac, long long max_rank, double zero_rel, double* __restrict__ thr_dev,
    long long* __restrict__ r_dev, double* __restrict__ Bm1, double* __restrict__ Bm2) {
  __shared__ int s_sk;
  if (threadIdx.x == 0) {
    const double l0 = lam[0];
    int nz = 0;
    for (int i = 0; i < m; ++i)
      if (lam[i] > zero_rel * l0 && lam[i] > 0.0) ++nz;
    if (nz == 0) nz = 1;
    int sk = nz;
    if (use_thr) {
      double thr;
      if (first) {
        double nrm2 = 0.0;
        for (int i = 0; i < m; ++i) nrm2 += fmax(lam[i], 0.0);
        thr = fac * sqrt(nrm2);
        *thr_dev = thr;
      } else {
        thr = *thr_dev;
      }
      double tail = 0.0;
      for (int i = nz - 1; i >= 1; --i) {
        tail += fmax(lam[i], 0.0);
        if (sqrt(tail) <= thr) sk = i; else break;
      }
      if (max_rank > 0 && sk > max_rank) sk = (int)max_rank;
    }
    s_sk = sk;
    if (r_dev) *r_dev = sk;
  }
  __syncthreads();
  const int sk = s_sk;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int c = e % m;
    double a = 0.0, b = 0.0;
    if (c < sk) {
      const double v = V[e];
      a = v * (1.0 / sqrt(fmax(lam[c], 1e-300)));
      b = v * sqrt(fmax(lam[c], 0.0));
    }
    Bm1[e] = a;
    Bm2[e] = b;
  }
}
__global__ void set_rank_kernel(long long* r_dev, long long idx, long long val) { r_dev[idx] = val; }

// Device-side decision of the accurate truncation (tt_round_async below the Gram floor): the
// unsorted singular values sg[0..kk) of the cluster Jacobi SVD are ranked by counting (the
// stable descending order of the host's std::stable_sort), then thread 0 applies the host
// loop's rule (numerical zeros sigma <= rk1 eps sigma_max, the delta tail, max_rank) with the
// same formulas and summation order.  perm[0..kk) = the sorted order, perm[kk] = the rank.
__global__ void __launch_bounds__(256) acc_decide_kernel(const double* __restrict__ sg, int kk,
                                                         int rk1, int first, double fac,
                                                         long long max_rank,
                                                         double* __restrict__ thr_dev,
                                                         long long* __restrict__ r_dev,
                                                         int* __restrict__ perm) {
  __shared__ int s_perm[256];
  __shared__ int s_sk;
  for (int i = threadIdx.x; i < kk; i += blockDim.x) {
    const double v = sg[i];
    int rk = 0;
    for (int j = 0; j < kk; ++j) rk += (sg[j] > v) || (sg[j] == v && j < i);
    s_perm[rk] = i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double thr;
    if (first) {
      double nrm2 = 0.0;
      for (int i = 0; i < kk; ++i) nrm2 += sg[i] * sg[i];
      thr = fac * sqrt(nrm2);
      *thr_dev = thr;
    } else {
      thr = *thr_dev;
    }
    const double smax = sg[s_perm[0]];
    int nz = 0;
    for (int i = 0; i < kk; ++i)
      if (sg[s_perm[i]] > (double)rk1 * 1.1e-16 * smax) ++nz;
    if (nz == 0) nz = 1;
    int sk = nz;
    double tail = 0.0;
    for (int i = nz - 1; i >= 1; --i) {
      tail += sg[s_perm[i]] * sg[s_perm[i]];
      if (sqrt(tail) <= thr) sk = i; else break;
    }
    if (max_rank > 0 && sk > max_rank) sk = (int)max_rank;
    s_sk = sk;
    *r_dev = sk;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kk; i += blockDim.x) perm[i] = s_perm[i];
  if (threadIdx.x == 0) perm[kk] = s_sk;
}
// the selected singular triplets zero-padded to the full width kk (rank = perm[kk]):
// Usel (kk x kk) = J[:, perm] with columns >= rank zero, SJt (kk x rk1) = (R^T J)[:, perm]^T
// with rows >= rank zero
__global__ void svd_select_padded_kernel(const double* __restrict__ BJ, const double* __restrict__ J,
                                         const int* __restrict__ perm, int kk, int rk1,
                                         double* __restrict__ Usel, double* __restrict__ SJt) {
  const int sk = perm[kk];
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < kk * kk) {
    const int r = e / kk, i = e - r * kk;
    Usel[e] = i < sk ? J[(long long)r * kk + perm[i]] : 0.0;
  }
  if (e < kk * rk1) {
    const int i = e / rk1, col = e - i * rk1;
    SJt[e] = i < sk ? BJ[(long long)col * kk + perm[i]] : 0.0;
  }
}

static tt_status round_impl(int64_t d, const int64_t* n, const int64_t* r_in,
                            const double* const* cores_in, double delta, int64_t max_rank,
                            int64_t* r_out, double* const* cores_out, void* workspace,
                            size_t workspace_bytes, void* stream, int phases, const char* who,
                            int64_t* r_dev = nullptr) {
  // r_dev != nullptr: asynchronous mode (tt_round_async) -- no host read of any singular value;
  // r_out receives the STORAGE ranks (host-known), r_dev (device) the effective ranks
  const bool async = r_dev != nullptr;
  if (d <= 0) return fail(TT_ERR_INVALID_ARGUMENT, "d must be >= 1");
  if (!n || !r_in || !cores_in || !r_out || !cores_out) return fail(TT_ERR_NULL_POINTER, "NULL array");
  if (r_in[0] != 1 || r_in[d] != 1) return fail(TT_ERR_INVALID_ARGUMENT, "r_1 and r_{d+1} must be 1");
  if (!(delta >= 0.0)) return fail(TT_ERR_INVALID_ARGUMENT, "delta must be >= 0");
  long long rmax = 0;
  for (int64_t k = 0; k < d; ++k) {
    if (n[k] <= 0 || r_in[k] <= 0) return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
    if (!cores_in[k] || !cores_out[k]) return fail(TT_ERR_NULL_POINTER, "NULL core");
    for (int64_t q = 0; q < d; ++q)
      if ((const void*)cores_out[k] == (const void*)cores_in[q])
        return fail(TT_ERR_ALIASING, "an output core aliases an input core");
    rmax = std::max<long long>(rmax, r_in[k]);
  }
  if (rmax > 512) return fail(TT_ERR_INVALID_ARGUMENT, "ranks above 512 are not supported");
  const size_t need = tt_round_workspace_size(d, n, r_in);
  if (need == 0) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Carver c{static_cast<char*>(workspace), workspace_bytes};
  std::vector<double*> W(d);
  long long core_max = 0;
  for (int64_t k = 0; k < d; ++k) {
    const long long sz = r_in[k] * n[k] * r_in[k + 1];
    W[k] = c.take(sz);
    core_max = std::max(core_max, sz);
  }
  double* Tmp = c.take(core_max);
  double* G = c.take(rmax * rmax);
  double* V = c.take(rmax * rmax);
  double* Bm = c.take(rmax * rmax);
  double* dg = c.take(rmax);
  double* lam = c.take(rmax);
  double* esc = c.take(sym_eigen_scratch(rmax));
  if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");
  std::vector<long long> r(r_in, r_in + d + 1);
  cudaError_t e = cudaSuccess;
  for (int64_t k = 0; k < d && e == cudaSuccess; ++k)
    e = cudaMemcpyAsync(W[k], cores_in[k], sizeof(double) * r[k] * n[k] * r[k + 1],
                        cudaMemcpyDeviceToDevice, s);
  std::vector<double> hl(rmax);
  // tt_round reads singular values on the host and returns synchronised; a pure cluster-QR
  // orthonormalisation (tt_orthonormalise with every unfolding on the QR path) reads nothing
  // and stays asynchronous
  bool host_sync = (phases & 2) != 0;
  auto eig = [&](int m) -> cudaError_t {   // G (m x m) -> V, lam (host copy in hl)
    host_sync = true;
    cudaError_t er = launch_sym_eigen(G, V, lam, m, esc, s);
    if (er != cudaSuccess) return er;
    er = cudaMemcpyAsync(hl.data(), lam, sizeof(double) * m, cudaMemcpyDeviceToHost, s);
    if (er != cudaSuccess) return er;
    return cudaStreamSynchronize(s);
  };
  // scaled copies of the leading eigenvector columns: Bm[:, :s] = V[:, :s] * f
  std::vector<double> hf(rmax);
  auto scaled = [&](int m, int cols, const std::vector<double>& f) -> cudaError_t {
    cudaError_t er = cudaMemcpyAsync(dg, f.data(), sizeof(double) * cols, cudaMemcpyHostToDevice, s);
    if (er != cudaSuccess) return er;
    scale_cols_kernel<<<(m * cols + 255) / 256, 256, 0, s>>>(V, dg, Bm, m, cols);
    ++g_launches;
    return cudaGetLastError();
  };
  const double zero_rel = 1e-14;   // relative eigenvalue floor (numerical zero of the Gram)
  // right-to-left orthonormalisation by Householder QR (tt_qr.cuh, exact to working
  // precision): W_k^T = Q R, W_k <- Q^T, W_{k-1} <- W_{k-1} R^T.  The Gram route below remains
  // for unfoldings that do not fit one cluster's shared memory (debug bit 29 forces it).
  for (int64_t k = d - 1; (phases & 1) && k >= 1 && e == cudaSuccess; --k) {
    const long long rk = r[k], q = n[k] * r[k + 1];
    if (!(g_dbg_flags & (1 << 29)) && qr_fits((int)q, (int)rk)) {
      const long long kk = std::min(q, rk);
      QrArgs qa{};
      qa.M = W[k];
      qa.rs = 1;                 // M = W_k^T: M[i][j] = W_k[j][i]
      qa.cs = q;
      qa.m = (int)q;
      qa.c = (int)rk;
      qa.Q = W[k];               // new core = Q^T (kk x q), i.e. Q column-major
      qa.qrs = 1;
      qa.qcs = q;
      qa.R = G;                  // R (kk x rk)
      if ((e = launch_qr(qa, s)) != cudaSuccess) break;
      const long long m1 = r[k - 1] * n[k - 1];
      // W_{k-1} (m1 x kk) = W_{k-1} (m1 x rk) . R^T  (B[k'][n'] = R[n'][k']: K-contiguous)
      e = launch_gemm(true, true, gp(W[k - 1], rk, G, rk, Tmp, m1, kk, rk, tt::map_plain(kk),
                                     tt::map_plain(1)), s);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(W[k - 1], Tmp, sizeof(double) * m1 * kk, cudaMemcpyDeviceToDevice, s);
      r[k] = kk;
      continue;
    }
    g_stage = TT_ST_IL_S1;
    e = launch_gemm(true, true, gp(W[k], q, W[k], q, G, rk, rk, q, tt::map_plain(rk),
                                   tt::map_plain(1)), s);
    if (async) {   // full-size zero-padded factors, the rank stays on the device
      if (e == cudaSuccess) e = launch_sym_eigen(G, V, lam, (int)rk, esc, s);
      if (e != cudaSuccess) break;
      trunc_decide_kernel<<<1, 256, 0, s>>>(lam, V, (int)rk, 0, 0, 0.0, 0, zero_rel, dg, nullptr,
                                            Bm, G);
      ++g_launches;
      if ((e = cudaGetLastError()) != cudaSuccess) break;
      // Tmp (rk x q) = (V S^-1)^T W_k (rows >= rank zero)
      e = launch_gemm(false, false, gp(Bm, rk, W[k], q, Tmp, rk, q, rk, tt::map_plain(q),
                                       tt::map_plain(1)), s);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(W[k], Tmp, sizeof(double) * rk * q, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) break;
      const long long m1a = r[k - 1] * n[k - 1];
      e = launch_gemm(true, false, gp(W[k - 1], rk, G, rk, Tmp, m1a, rk, rk, tt::map_plain(rk),
                                      tt::map_plain(1)), s);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(W[k - 1], Tmp, sizeof(double) * m1a * rk, cudaMemcpyDeviceToDevice, s);
      continue;
    }
    if (e == cudaSuccess) e = eig((int)rk);
    if (e != cudaSuccess) break;
    int sk = 0;
    for (long long i = 0; i < rk; ++i)
      if (hl[i] > zero_rel * hl[0] && hl[i] > 0.0) ++sk;
    if (sk == 0) sk = 1;
    for (int i = 0; i < sk; ++i) hf[i] = 1.0 / std::sqrt(std::max(hl[i], 1e-300));
    if ((e = scaled((int)rk, sk, hf)) != cudaSuccess) break;
    // Tmp (sk x q) = (V S^-1)^T W_k
    e = launch_gemm(false, false, gp(Bm, sk, W[k], q, Tmp, sk, q, rk, tt::map_plain(q),
                                     tt::map_plain(1)), s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(W[k], Tmp, sizeof(double) * sk * q, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) break;
    for (int i = 0; i < sk; ++i) hf[i] = std::sqrt(std::max(hl[i], 0.0));
    if ((e = scaled((int)rk, sk, hf)) != cudaSuccess) break;
    // W_{k-1} (r_{k-1} n x sk) = W_{k-1} (r_{k-1} n x rk) . (V S)
    const long long m1 = r[k - 1] * n[k - 1];
    e = launch_gemm(true, false, gp(W[k - 1], rk, Bm, sk, Tmp, m1, sk, rk, tt::map_plain(sk),
                                    tt::map_plain(1)), s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(W[k - 1], Tmp, sizeof(double) * m1 * sk, cudaMemcpyDeviceToDevice, s);
    r[k] = sk;
  }
  // left orthonormalisation without truncation (tt_orthonormalise, phases bit 4): Householder
  // QR W_k = Q R, W_k <- Q, W_{k+1} <- R W_{k+1}
  for (int64_t k = 0; (phases & 4) && k < d - 1 && e == cudaSuccess; ++k) {
    const long long m = r[k] * n[k], rk1 = r[k + 1];
    if ((g_dbg_flags & (1 << 29)) || !qr_fits((int)m, (int)rk1)) {   // Gram route for this core
      phases |= 2;
      break;
    }
    const long long kk = std::min(m, rk1);
    QrArgs qa{};
    qa.M = W[k];
    qa.rs = rk1;
    qa.cs = 1;
    qa.m = (int)m;
    qa.c = (int)rk1;
    qa.Q = W[k];   // Q (m x kk) row-major
    qa.qrs = kk;
    qa.qcs = 1;
    qa.R = G;
    if ((e = launch_qr(qa, s)) != cudaSuccess) break;
    const long long q = n[k + 1] * r[k + 2];
    // W_{k+1} (kk x q) = R (kk x rk1) . W_{k+1} (rk1 x q)
    e = launch_gemm(true, false, gp(G, rk1, W[k + 1], q, Tmp, kk, q, rk1, tt::map_plain(q),
                                    tt::map_plain(1)), s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(W[k + 1], Tmp, sizeof(double) * kk * q, cudaMemcpyDeviceToDevice, s);
    r[k + 1] = kk;
  }
  // left-to-right truncation with threshold delta / sqrt(d-1) ||T||
  double thr = 0.0;
  // Accurate route (Householder QR + one-sided Jacobi SVD of R^T, no squared-condition floor;
  // Jacobi on R^T rather than R converges in ~8 sweeps at any condition, as in LAPACK's
  // preconditioned dgejsv, where R's own columns need 11-26+ growing with the condition)
  // where the Gram route's floor (singular values below ~1e-8 sigma_max unresolved) reaches the
  // per-core threshold: delta / sqrt(d-1) < 1e-7, delta = 0 included; debug bit 24 forces it.
  const bool accurate = (phases & 2) &&
      ((g_dbg_flags & (1 << 24)) || delta / std::sqrt((double)std::max<int64_t>(d - 1, 1)) < 1e-7);
  int64_t kstart = 0;   // the Gram route continues from the first core the accurate one left
  for (int64_t k = 0; accurate && k < d - 1 && e == cudaSuccess; ++k) {
    const long long m = r[k] * n[k], rk1 = r[k + 1], kk = std::min(m, rk1);
    if (!qr_fits((int)m, (int)rk1) || !svd_fits((int)rk1, (int)kk)) break;   // Gram from here
    QrArgs qa{};
    qa.M = W[k];
    qa.rs = rk1;
    qa.cs = 1;
    qa.m = (int)m;
    qa.c = (int)rk1;
    qa.Q = W[k];   // Q (m x kk) row-major
    qa.qrs = kk;
    qa.qcs = 1;
    qa.R = G;      // R (kk x rk1)
    if ((e = launch_qr(qa, s)) != cudaSuccess) break;
    SvdArgs sa{};
    sa.B = G;      // R (kk x rk1) row-major = R^T (rk1 x kk) column-major
    sa.bt = 1;
    sa.rows = (int)rk1;
    sa.c = (int)kk;
    sa.BJ = Bm;    // R^T J (rk1 x kk)
    sa.J = V;      // J (kk x kk)
    sa.sigma = lam;
    sa.sweeps = nullptr;
    if ((e = launch_svd(sa, s)) != cudaSuccess) break;
    if (async) {   // rank, order and selection on the device; every extent stays kk
      double* Usel = esc;
      double* SJt = esc + rmax * rmax;
      int* dperm = reinterpret_cast<int*>(esc + 2 * rmax * rmax);
      const double fac = delta / std::sqrt((double)std::max<int64_t>(d - 1, 1));
      acc_decide_kernel<<<1, 256, 0, s>>>(lam, (int)kk, (int)rk1, k == 0 ? 1 : 0, fac,
                                          (long long)max_rank, dg,
                                          reinterpret_cast<long long*>(r_dev) + k + 1, dperm);
      const long long nsel = std::max(kk, rk1) * kk;
      svd_select_padded_kernel<<<(unsigned)((nsel + 255) / 256), 256, 0, s>>>(
          Bm, V, dperm, (int)kk, (int)rk1, Usel, SJt);
      g_launches += 2;
      if ((e = cudaGetLastError()) != cudaSuccess) break;
      e = launch_gemm(true, false, gp(W[k], kk, Usel, kk, Tmp, m, kk, kk, tt::map_plain(kk),
                                      tt::map_plain(1)), s);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(W[k], Tmp, sizeof(double) * m * kk, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) break;
      const long long qa3 = n[k + 1] * r[k + 2];
      e = launch_gemm(true, false, gp(SJt, rk1, W[k + 1], qa3, Tmp, kk, qa3, rk1, tt::map_plain(qa3),
                                      tt::map_plain(1)), s);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(W[k + 1], Tmp, sizeof(double) * kk * qa3, cudaMemcpyDeviceToDevice, s);
      r[k + 1] = kk;
      kstart = k + 1;
      continue;
    }
    std::vector<double> sg(kk);
    if ((e = cudaMemcpyAsync(sg.data(), lam, sizeof(double) * kk, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaStreamSynchronize(s)) != cudaSuccess)
      break;
    std::vector<int> perm(kk);
    for (int i = 0; i < (int)kk; ++i) perm[i] = i;
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return sg[a] > sg[b]; });
    if (k == 0) {
      double nrm2 = 0.0;
      for (long long i = 0; i < kk; ++i) nrm2 += sg[i] * sg[i];
      thr = delta / std::sqrt((double)std::max<int64_t>(d - 1, 1)) * std::sqrt(nrm2);
    }
    // numerical zeros: sigma <= rk1 eps sigma_max (the QR's backward error)
    const double smax = sg[perm[0]];
    int nz = 0;
    for (long long i = 0; i < kk; ++i)
      if (sg[perm[i]] > (double)rk1 * 1.1e-16 * smax) ++nz;
    if (nz == 0) nz = 1;
    int sk = nz;
    double tail = 0.0;
    for (int i = nz - 1; i >= 1; --i) {
      tail += sg[perm[i]] * sg[perm[i]];
      if (std::sqrt(tail) <= thr) sk = i; else break;
    }
    if (max_rank > 0 && sk > max_rank) sk = (int)max_rank;
    // Usel (kk x sk) = J[:, perm], SJt (sk x rk1) = (R^T J)[:, perm]^T = sigma U_R^T
    double* Usel = esc;
    double* SJt = esc + rmax * rmax;
    int* dperm = reinterpret_cast<int*>(esc + 2 * rmax * rmax);
    if ((e = cudaMemcpyAsync(dperm, perm.data(), sizeof(int) * sk, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      break;
    const long long nsel = std::max(kk, rk1) * sk;
    svd_select_kernel<<<(unsigned)((nsel + 255) / 256), 256, 0, s>>>(Bm, V, dperm, (int)kk,
                                                                      (int)rk1, sk, Usel, SJt);
    ++g_launches;
    if ((e = cudaGetLastError()) != cudaSuccess) break;
    // new core (m x sk) = Q (m x kk) . Usel
    e = launch_gemm(true, false, gp(W[k], kk, Usel, sk, Tmp, m, sk, kk, tt::map_plain(sk),
                                    tt::map_plain(1)), s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(W[k], Tmp, sizeof(double) * m * sk, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) break;
    // W_{k+1} (sk x q) = SJt (sk x rk1) . W_{k+1} (rk1 x q)
    const long long q = n[k + 1] * r[k + 2];
    e = launch_gemm(true, false, gp(SJt, rk1, W[k + 1], q, Tmp, sk, q, rk1, tt::map_plain(q),
                                    tt::map_plain(1)), s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(W[k + 1], Tmp, sizeof(double) * sk * q, cudaMemcpyDeviceToDevice, s);
    r[k + 1] = sk;
    kstart = k + 1;
  }
  for (int64_t k = kstart; (phases & 2) && k < d - 1 && e == cudaSuccess; ++k) {
    const long long m = r[k] * n[k], rk1 = r[k + 1];
    g_stage = TT_ST_IL_S2;
    e = launch_gemm(false, false, gp(W[k], rk1, W[k], rk1, G, rk1, rk1, m, tt::map_plain(rk1),
                                     tt::map_plain(1)), s);
    if (async) {   // device-side rank decision, full-size zero-padded update GEMMs
      if (e == cudaSuccess) e = launch_sym_eigen(G, V, lam, (int)rk1, esc, s);
      if (e != cudaSuccess) break;
      const double fac = delta / std::sqrt((double)std::max<int64_t>(d - 1, 1));
      trunc_decide_kernel<<<1, 256, 0, s>>>(lam, V, (int)rk1, 1, k == 0 ? 1 : 0, fac,
                                            (long long)max_rank, zero_rel, dg,
                                            reinterpret_cast<long long*>(r_dev) + k + 1, Bm, G);
      ++g_launches;
      if ((e = cudaGetLastError()) != cudaSuccess) break;
      // U (m x rk1) = W_k . (V S^-1) (columns >= rank zero)
      e = launch_gemm(true, false, gp(W[k], rk1, Bm, rk1, Tmp, m, rk1, rk1, tt::map_plain(rk1),
                                      tt::map_plain(1)), s);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(W[k], Tmp, sizeof(double) * m * rk1, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) break;
      // W_{k+1} (rk1 x q) = (V S)^T . W_{k+1} (rows >= rank zero)
      const long long qa2 = n[k + 1] * r[k + 2];
      e = launch_gemm(false, false, gp(G, rk1, W[k + 1], qa2, Tmp, rk1, qa2, rk1, tt::map_plain(qa2),
                                       tt::map_plain(1)), s);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(W[k + 1], Tmp, sizeof(double) * rk1 * qa2, cudaMemcpyDeviceToDevice, s);
      continue;
    }
    if (e == cudaSuccess) e = eig((int)rk1);
    if (e != cudaSuccess) break;
    if (k == 0) {
      double nrm2 = 0.0;
      for (long long i = 0; i < rk1; ++i) nrm2 += std::max(hl[i], 0.0);
      thr = delta / std::sqrt((double)std::max<int64_t>(d - 1, 1)) * std::sqrt(nrm2);
    }
    // smallest rank whose discarded tail has Frobenius norm <= thr; drop numerical zeros
    int nz = 0;
    for (long long i = 0; i < rk1; ++i)
      if (hl[i] > zero_rel * hl[0] && hl[i] > 0.0) ++nz;
    if (nz == 0) nz = 1;
    int sk = nz;
    double tail = 0.0;
    for (int i = nz - 1; i >= 1; --i) {
      tail += std::max(hl[i], 0.0);
      if (std::sqrt(tail) <= thr) sk = i; else break;
    }
    if (max_rank > 0 && sk > max_rank) sk = (int)max_rank;
    for (int i = 0; i < sk; ++i) hf[i] = 1.0 / std::sqrt(std::max(hl[i], 1e-300));
    if ((e = scaled((int)rk1, sk, hf)) != cudaSuccess) break;
    // U (m x sk) = W_k . (V S^-1)
    e = launch_gemm(true, false, gp(W[k], rk1, Bm, sk, Tmp, m, sk, rk1, tt::map_plain(sk),
                                    tt::map_plain(1)), s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(W[k], Tmp, sizeof(double) * m * sk, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) break;
    for (int i = 0; i < sk; ++i) hf[i] = std::sqrt(std::max(hl[i], 0.0));
    if ((e = scaled((int)rk1, sk, hf)) != cudaSuccess) break;
    // W_{k+1} (sk x q) = (V S)^T . W_{k+1} (rk1 x q)
    const long long q = n[k + 1] * r[k + 2];
    e = launch_gemm(false, false, gp(Bm, sk, W[k + 1], q, Tmp, sk, q, rk1, tt::map_plain(q),
                                     tt::map_plain(1)), s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(W[k + 1], Tmp, sizeof(double) * sk * q, cudaMemcpyDeviceToDevice, s);
    r[k + 1] = sk;
  }
  for (int64_t k = 0; k < d && e == cudaSuccess; ++k)
    e = cudaMemcpyAsync(cores_out[k], W[k], sizeof(double) * r[k] * n[k] * r[k + 1],
                        cudaMemcpyDeviceToDevice, s);
  if (async && e == cudaSuccess) {
    set_rank_kernel<<<1, 1, 0, s>>>(reinterpret_cast<long long*>(r_dev), 0, 1);
    set_rank_kernel<<<1, 1, 0, s>>>(reinterpret_cast<long long*>(r_dev), d, 1);
    g_launches += 2;
    e = cudaGetLastError();
  } else if (e == cudaSuccess && (host_sync || (phases & 2))) {
    e = cudaStreamSynchronize(s);
  }
  if (e != cudaSuccess) return cuda_fail(e, who);
  for (int64_t k = 0; k <= d; ++k) r_out[k] = r[k];
  return TT_OK;
}

tt_status tt_round(int64_t d, const int64_t* n, const int64_t* r_in,
                   const double* const* cores_in, double delta, int64_t max_rank, int64_t* r_out,
                   double* const* cores_out, void* workspace, size_t workspace_bytes,
                   void* stream) {
  CallScope scope;
  return round_impl(d, n, r_in, cores_in, delta, max_rank, r_out, cores_out, workspace,
                    workspace_bytes, stream, 3, "tt_round");
}

tt_status tt_round_async(int64_t d, const int64_t* n, const int64_t* r_in,
                         const double* const* cores_in, double delta, int64_t max_rank,
                         int64_t* r_storage, int64_t* r_dev, double* const* cores_out,
                         void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  if (!r_dev) return fail(TT_ERR_NULL_POINTER, "r_dev is NULL");
  return round_impl(d, n, r_in, cores_in, delta, max_rank, r_storage, cores_out, workspace,
                    workspace_bytes, stream, 3, "tt_round_async", r_dev);
}

size_t tt_orthonormalise_workspace_size(int64_t d, const int64_t* n, const int64_t* r) {
  return tt_round_workspace_size(d, n, r);
}

tt_status tt_orthonormalise(int64_t d, const int64_t* n, const int64_t* r_in,
                            const double* const* cores_in, int direction, int64_t* r_out,
                            double* const* cores_out, void* workspace, size_t workspace_bytes,
                            void* stream) {
  CallScope scope;
  if (direction != TT_SWEEP_LEFT && direction != TT_SWEEP_RIGHT)
    return fail(TT_ERR_INVALID_ARGUMENT, "direction must be TT_SWEEP_LEFT or TT_SWEEP_RIGHT");
  return round_impl(d, n, r_in, cores_in, 0.0, 0, r_out, cores_out, workspace, workspace_bytes,
                    stream, direction == TT_SWEEP_LEFT ? 4 : 1, "tt_orthonormalise");
}

tt_status tt_debug_svd(int64_t rows, int64_t c, const double* B, double* BJ, double* J,
                       double* sigma, int32_t* sweeps, void* stream) {
  CallScope scope;
  if (rows <= 0 || c <= 0) return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  if (!B || !BJ || !J || !sigma) return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  if (!svd_fits((int)rows, (int)c)) return fail(TT_ERR_INVALID_ARGUMENT, "rows, c <= 256");
  SvdArgs a{};
  a.B = B;
  a.rows = (int)rows;
  a.c = (int)c;
  a.BJ = BJ;
  a.J = J;
  a.sigma = sigma;
  a.sweeps = reinterpret_cast<int*>(sweeps);
  cudaError_t e = launch_svd(a, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tt_debug_svd");
  return TT_OK;
}

// ---- block-index move ---------------------------------
// Thin SVD of an m x q matrix M through the Gram matrix of its smaller side: the leading s
// left singular vectors Us (m x s) and right singular vectors Vs (q x s), truncated at
// ||sigma_{s:}|| <= delta ||sigma|| (numerical zeros lambda <= 1e-14 lambda_max dropped) and
// s <= max_rank.  One host synchronisation (the truncation is data dependent).
struct SvdBufs {
  double *G, *E, *lam, *esc, *f, *Us, *Vs;
};
static long long svd_ws_elems(long long m, long long q) {
  const long long k = std::min(m, q), big = std::max(m, q);
  // G, E (<= k^2 + big k), lam, eigen scratch, f, Us + Vs (<= 2 big k), alignment slack
  return 2 * k * k + 3 * big * k + 3 * k + 128 + sym_eigen_scratch(k) + 12 * 32;
}
// Device-side truncation decision of the asynchronous block moves: the rule of svd_gram's
// host loop (same formulas and summation order) from the descending Gram eigenvalues; writes
// the rank and the column factors 1 / sigma (0 beyond the rank); svd_mask_kernel then zeroes
// the columns >= rank of the Gram side's singular vectors, so every later GEMM keeps extent k.
__global__ void __launch_bounds__(256) svd_decide_kernel(const double* __restrict__ lam, int k,
                                                         double delta, long long max_rank,
                                                         long long* __restrict__ s_dev,
                                                         double* __restrict__ fin) {
  __shared__ int s_sk;
  if (threadIdx.x == 0) {
    double tot = 0.0;
    int nz = 0;
    for (int i = 0; i < k; ++i) {
      tot += fmax(lam[i], 0.0);
      if (lam[i] > 1e-14 * lam[0] && lam[i] > 0.0) ++nz;
    }
    if (nz == 0) nz = 1;
    const double thr = delta * sqrt(tot);
    int sk = nz;
    double tail = 0.0;
    for (int i = nz - 1; i >= 1; --i) {
      tail += fmax(lam[i], 0.0);
      if (sqrt(tail) <= thr) sk = i; else break;
    }
    if (max_rank > 0 && sk > max_rank) sk = (int)max_rank;
    s_sk = sk;
    *s_dev = sk;
  }
  __syncthreads();
  const int sk = s_sk;
  for (int c = threadIdx.x; c < k; c += blockDim.x)
    fin[c] = c < sk ? 1.0 / sqrt(fmax(lam[c], 1e-300)) : 0.0;
}
// side = E with the columns >= *s_dev zeroed (k x k, all SMs)
__global__ void svd_mask_kernel(const double* __restrict__ E, int k,
                                const long long* __restrict__ s_dev, double* __restrict__ side) {
  const int sk = (int)*s_dev;
  const long long kk = (long long)k * k;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < kk;
       e += (long long)gridDim.x * blockDim.x)
    side[e] = (int)(e % k) < sk ? E[e] : 0.0;
}

static cudaError_t svd_gram(const double* M, long long m, long long q, double delta,
                            long long max_rank, SvdBufs& b, int& s_out, cudaStream_t s,
                            int64_t* s_dev = nullptr) {
  const bool left = m <= q;   // Gram of the smaller side
  const long long k = left ? m : q;
  cudaError_t e;
  g_stage = TT_ST_IL_S1;
  if (left)   // G = M M^T (m x m)
    e = launch_gemm(true, true, gp(M, q, M, q, b.G, m, m, q, tt::map_plain(m), tt::map_plain(1)), s);
  else        // G = M^T M (q x q)
    e = launch_gemm(false, false, gp(M, q, M, q, b.G, q, q, m, tt::map_plain(q), tt::map_plain(1)), s);
  if (e != cudaSuccess) return e;
  if ((e = launch_sym_eigen(b.G, b.E, b.lam, (int)k, b.esc, s)) != cudaSuccess) return e;
  if (s_dev) {   // asynchronous: rank on the device, every extent stays k (zero padding)
    double* side = left ? b.Us : b.Vs;
    double* fin = b.f + 32 * ((k + 31) / 32);
    svd_decide_kernel<<<1, 256, 0, s>>>(b.lam, (int)k, delta, max_rank,
                                        reinterpret_cast<long long*>(s_dev), fin);
    svd_mask_kernel<<<(unsigned)std::min<long long>(4096, (k * k + 255) / 256), 256, 0, s>>>(
        b.E, (int)k, reinterpret_cast<const long long*>(s_dev), side);
    g_launches += 2;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    s_out = (int)k;
    double* other = left ? b.Vs : b.Us;
    if (left)   // Vs (q x k) = M^T (q x m) . Us (m x k)
      e = launch_gemm(false, false, gp(M, q, b.Us, k, b.E, q, k, m, tt::map_plain(k), tt::map_plain(1)), s);
    else        // Us (m x k) = M (m x q) . Vs (q x k)
      e = launch_gemm(true, false, gp(M, q, b.Vs, k, b.E, m, k, q, tt::map_plain(k), tt::map_plain(1)), s);
    if (e != cudaSuccess) return e;
    const long long ob = left ? q : m;
    scale_cols_ld_kernel<<<(unsigned)std::min<long long>(4096, (ob * k + 255) / 256), 256, 0, s>>>(
        b.E, k, fin, other, ob, (int)k);
    ++g_launches;
    return cudaGetLastError();
  }
  std::vector<double> hl(k);
  if ((e = cudaMemcpyAsync(hl.data(), b.lam, sizeof(double) * k, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  double tot = 0.0;
  int nz = 0;
  for (long long i = 0; i < k; ++i) {
    tot += std::max(hl[i], 0.0);
    if (hl[i] > 1e-14 * hl[0] && hl[i] > 0.0) ++nz;
  }
  if (nz == 0) nz = 1;
  const double thr = delta * std::sqrt(tot);
  int sk = nz;
  double tail = 0.0;
  for (int i = nz - 1; i >= 1; --i) {
    tail += std::max(hl[i], 0.0);
    if (std::sqrt(tail) <= thr) sk = i; else break;
  }
  if (max_rank > 0 && sk > max_rank) sk = (int)max_rank;
  s_out = sk;
  // E[:, :sk] (k x sk) -> the singular vectors of the Gram side; the other side by a GEMM
  std::vector<double> hf(sk);
  for (int i = 0; i < sk; ++i) hf[i] = 1.0;
  if ((e = cudaMemcpyAsync(b.f, hf.data(), sizeof(double) * sk, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return e;
  double* side = left ? b.Us : b.Vs;
  scale_cols_kernel<<<(unsigned)((k * sk + 255) / 256), 256, 0, s>>>(b.E, b.f, side, (int)k, sk);
  ++g_launches;
  for (int i = 0; i < sk; ++i) hf[i] = 1.0 / std::sqrt(std::max(hl[i], 1e-300));
  double* fin = b.f + 32 * ((sk + 31) / 32);
  if ((e = cudaMemcpyAsync(fin, hf.data(), sizeof(double) * sk, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return e;
  // the other side: Vs = M^T Us Sigma^-1  or  Us = M Vs Sigma^-1 (scale columns afterwards)
  double* other = left ? b.Vs : b.Us;
  if (left)   // Vs (q x sk) = M^T (q x m) . Us (m x sk)
    e = launch_gemm(false, false, gp(M, q, b.Us, sk, b.E, q, sk, m, tt::map_plain(sk), tt::map_plain(1)), s);
  else        // Us (m x sk) = M (m x q) . Vs (q x sk)
    e = launch_gemm(true, false, gp(M, q, b.Vs, sk, b.E, m, sk, q, tt::map_plain(sk), tt::map_plain(1)), s);
  if (e != cudaSuccess) return e;
  const long long ob = left ? q : m;
  scale_cols_ld_kernel<<<(unsigned)std::min<long long>(4096, (ob * sk + 255) / 256), 256, 0, s>>>(
      b.E, sk, fin, other, ob, sk);
  ++g_launches;
  return cudaGetLastError();
}

static bool block_move_ws(long long m, long long q, long long extra, long long& total) {
  total = svd_ws_elems(m, q) + m * q + extra;
  return m > 0 && q > 0;
}

size_t tt_block_move_workspace_size(int64_t r0, int64_t n0, int64_t l, int64_t r1, int64_t n1,
                                    int64_t r2) {
  if (r0 <= 0 || n0 <= 0 || l <= 0 || r1 <= 0 || n1 <= 0 || r2 <= 0) return 0;
  bool ok = true;
  // right move: M = (r0 n0) x (l r1);  left move: M = (r0 l) x (n0 r1) with (r0,n0,l,r1) the
  // core carrying the block index -- size for the larger of the two views
  const long long m1 = prod({r0, n0}, ok), q1 = prod({l, r1}, ok);
  const long long m2 = prod({r1, l}, ok), q2 = prod({n1, r2}, ok);
  const long long out = prod({std::max(m1, q1), std::max(n1 * r2, r0 * n0), l}, ok);
  if (!ok) return 0;
  long long a, b;
  block_move_ws(m1, q1, out, a);
  block_move_ws(m2, q2, out, b);
  return ws_bytes({std::max(a, b)});
}

static tt_status block_move_right_impl(int64_t r0, int64_t n0, int64_t l, int64_t r1, int64_t n1,
                              int64_t r2, double delta, int64_t max_rank, const double* Wk_hat,
                              const double* Wk1, double* Wk_out, double* Wk1_hat_out,
                              int64_t* s_out, void* workspace, size_t workspace_bytes,
                              void* stream, int64_t* s_dev) {
  if (r0 <= 0 || n0 <= 0 || l <= 0 || r1 <= 0 || n1 <= 0 || r2 <= 0)
    return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  if (!(delta >= 0.0) || max_rank < 0) return fail(TT_ERR_INVALID_ARGUMENT, "need delta >= 0, max_rank >= 0");
  if (!Wk_hat || !Wk1 || !Wk_out || !Wk1_hat_out || !s_out) return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  for (const void* o : {(const void*)Wk_out, (const void*)Wk1_hat_out})
    if (same(o, Wk_hat) || same(o, Wk1)) return fail(TT_ERR_ALIASING, "an output aliases an input");
  if (same(Wk_out, Wk1_hat_out)) return fail(TT_ERR_ALIASING, "two outputs alias");
  const long long m = r0 * n0, q = l * r1;
  if (std::min(m, q) > 2048)
    return fail(TT_ERR_INVALID_ARGUMENT, "min(r0 n0, l r1) above 2048 is not supported");
  const size_t need = tt_block_move_workspace_size(r0, n0, l, r1, n1, r2);
  if (need == 0) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long k = std::min(m, q), big = std::max(m, q);
  Carver c{static_cast<char*>(workspace), workspace_bytes};
  SvdBufs b;
  b.G = c.take(k * k);
  b.E = c.take(std::max(k * k, big * k));
  b.lam = c.take(k);
  b.esc = c.take(sym_eigen_scratch(k));
  b.f = c.take(2 * (k + 64));
  b.Us = c.take(m * k);
  b.Vs = c.take(q * k);
  double* C = c.take(k * q);
  if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");
  int sk = 0;
  cudaError_t e = svd_gram(Wk_hat, m, q, delta, max_rank, b, sk, s, s_dev);
  // Wk_out = Us (m x sk);  C (sk x q) = Us^T M
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(Wk_out, b.Us, sizeof(double) * m * sk, cudaMemcpyDeviceToDevice, s);
  g_stage = TT_ST_IL_S2;
  if (e == cudaSuccess)
    e = launch_gemm(false, false, gp(b.Us, sk, Wk_hat, q, C, sk, q, m, tt::map_plain(q),
                                     tt::map_plain(1)), s);
  // Wk1_hat_out[s, j, l, c] = sum_b C[s, l, b] Wk1[b, j, c]: rows (s, l), cols (j, c)
  if (e == cudaSuccess)
    e = launch_gemm(true, false, gp(C, r1, Wk1, n1 * r2, Wk1_hat_out, sk * l, n1 * r2, r1,
                                    tt::map2(l, r2, n1 * l * r2), tt::map2(r2, 1, l * r2)), s);
  if (e == cudaSuccess && !s_dev) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "tt_block_move_right");
  *s_out = sk;
  return TT_OK;
}
tt_status tt_block_move_right(int64_t r0, int64_t n0, int64_t l, int64_t r1, int64_t n1,
                              int64_t r2, double delta, int64_t max_rank, const double* Wk_hat,
                              const double* Wk1, double* Wk_out, double* Wk1_hat_out,
                              int64_t* s_out, void* workspace, size_t workspace_bytes,
                              void* stream) {
  CallScope scope;
  return block_move_right_impl(r0, n0, l, r1, n1, r2, delta, max_rank, Wk_hat, Wk1, Wk_out,
                               Wk1_hat_out, s_out, workspace, workspace_bytes, stream, nullptr);
}
tt_status tt_block_move_right_async(int64_t r0, int64_t n0, int64_t l, int64_t r1, int64_t n1,
                                    int64_t r2, double delta, int64_t max_rank,
                                    const double* Wk_hat, const double* Wk1, double* Wk_out,
                                    double* Wk1_hat_out, int64_t* s_storage, int64_t* s_dev,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  if (!s_dev) return fail(TT_ERR_NULL_POINTER, "s_dev is NULL");
  return block_move_right_impl(r0, n0, l, r1, n1, r2, delta, max_rank, Wk_hat, Wk1, Wk_out,
                               Wk1_hat_out, s_storage, workspace, workspace_bytes, stream, s_dev);
}

static tt_status block_move_left_impl(int64_t r0, int64_t n0, int64_t r1, int64_t n1, int64_t l,
                             int64_t r2, double delta, int64_t max_rank, const double* Wkm1,
                             const double* Wk_hat, double* Wkm1_hat_out, double* Wk_out,
                             int64_t* s_out, void* workspace, size_t workspace_bytes,
                             void* stream, int64_t* s_dev) {
  if (r0 <= 0 || n0 <= 0 || l <= 0 || r1 <= 0 || n1 <= 0 || r2 <= 0)
    return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  if (!(delta >= 0.0) || max_rank < 0) return fail(TT_ERR_INVALID_ARGUMENT, "need delta >= 0, max_rank >= 0");
  if (!Wkm1 || !Wk_hat || !Wk_out || !Wkm1_hat_out || !s_out) return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  for (const void* o : {(const void*)Wk_out, (const void*)Wkm1_hat_out})
    if (same(o, Wk_hat) || same(o, Wkm1)) return fail(TT_ERR_ALIASING, "an output aliases an input");
  if (same(Wk_out, Wkm1_hat_out)) return fail(TT_ERR_ALIASING, "two outputs alias");
  const long long m = r1 * l, q = n1 * r2;
  if (std::min(m, q) > 2048)
    return fail(TT_ERR_INVALID_ARGUMENT, "min(r1 l, n1 r2) above 2048 is not supported");
  const size_t need = tt_block_move_workspace_size(r0, n0, l, r1, n1, r2);
  if (need == 0) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long k = std::min(m, q), big = std::max(m, q);
  Carver c{static_cast<char*>(workspace), workspace_bytes};
  SvdBufs b;
  b.G = c.take(k * k);
  b.E = c.take(std::max(k * k, big * k));
  b.lam = c.take(k);
  b.esc = c.take(sym_eigen_scratch(k));
  b.f = c.take(2 * (k + 64));
  b.Us = c.take(m * k);
  b.Vs = c.take(q * k);
  double* Mp = c.take(m * q);
  double* C = c.take(m * k);
  if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");
  long long blocks = std::min<long long>(4096, (m * q + 255) / 256);
  // M (r1 l) x (n1 r2) from Wk_hat (r1, n1, l, r2)
  swap_mid_kernel<<<(unsigned)blocks, 256, 0, s>>>(Wk_hat, Mp, r1, n1, l, r2);
  ++g_launches;
  int sk = 0;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = svd_gram(Mp, m, q, delta, max_rank, b, sk, s, s_dev);
  // Wk_out (sk x q) = Vs^T;  C (m x sk) = M Vs = Us Sigma
  if (e == cudaSuccess) {
    transpose2d_kernel<<<(unsigned)std::min<long long>(4096, (q * sk + 255) / 256), 256, 0, s>>>(
        b.Vs, Wk_out, q, sk);
    ++g_launches;
    e = cudaGetLastError();
  }
  g_stage = TT_ST_IL_S2;
  if (e == cudaSuccess)
    e = launch_gemm(true, false, gp(Mp, q, b.Vs, sk, C, m, sk, q, tt::map_plain(sk),
                                    tt::map_plain(1)), s);
  // Wkm1_hat_out (r0 n0) x (l sk) = Wkm1 (r0 n0 x r1) . C (r1 x (l sk))
  if (e == cudaSuccess)
    e = launch_gemm(true, false, gp(Wkm1, r1, C, l * sk, Wkm1_hat_out, r0 * n0, l * sk, r1,
                                    tt::map_plain(l * sk), tt::map_plain(1)), s);
  if (e == cudaSuccess && !s_dev) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "tt_block_move_left");
  *s_out = sk;
  return TT_OK;
}
tt_status tt_block_move_left(int64_t r0, int64_t n0, int64_t r1, int64_t n1, int64_t l,
                             int64_t r2, double delta, int64_t max_rank, const double* Wkm1,
                             const double* Wk_hat, double* Wkm1_hat_out, double* Wk_out,
                             int64_t* s_out, void* workspace, size_t workspace_bytes,
                             void* stream) {
  CallScope scope;
  return block_move_left_impl(r0, n0, r1, n1, l, r2, delta, max_rank, Wkm1, Wk_hat, Wkm1_hat_out,
                              Wk_out, s_out, workspace, workspace_bytes, stream, nullptr);
}
tt_status tt_block_move_left_async(int64_t r0, int64_t n0, int64_t r1, int64_t n1, int64_t l,
                                   int64_t r2, double delta, int64_t max_rank, const double* Wkm1,
                                   const double* Wk_hat, double* Wkm1_hat_out, double* Wk_out,
                                   int64_t* s_storage, int64_t* s_dev, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  CallScope scope;
  if (!s_dev) return fail(TT_ERR_NULL_POINTER, "s_dev is NULL");
  return block_move_left_impl(r0, n0, r1, n1, l, r2, delta, max_rank, Wkm1, Wk_hat, Wkm1_hat_out,
                              Wk_out, s_storage, workspace, workspace_bytes, stream, s_dev);
}

// ---- AMEn enrichment ("enrichment of the TT cores by TT cores of the
// approximate residual, as in the AMEn algorithm") -----------------------------------------
// x_k (rl, n, rx) and the residual core z_k (rl, n, rz) are concatenated along the right bond,
// x_{k+1} (rx, n1, r2) is padded with rz zero rows (the represented tensor is unchanged), and
// the enlarged core is re-orthonormalised by one truncated SVD step (tt_block_move_right with
// l = 1): x_k' (rl, n, s) left-orthonormal, x_{k+1}' (s, n1, r2).
__global__ void enrich_concat_kernel(const double* __restrict__ x, const double* __restrict__ z,
                                     const double* __restrict__ x1, double* __restrict__ cat,
                                     double* __restrict__ cat1, long long rows, long long rx,
                                     long long rz, long long q1) {
  const long long r = rx + rz;
  const long long n0 = rows * r, n1 = r * q1;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n0 + n1;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < n0) {
      const long long i = e / r, c = e - i * r;
      cat[e] = c < rx ? x[i * rx + c] : z[i * rz + (c - rx)];
    } else {
      const long long f = e - n0, row = f / q1;
      cat1[f] = row < rx ? x1[f] : 0.0;
    }
  }
}

size_t tt_enrich_right_workspace_size(int64_t rl, int64_t n, int64_t rx, int64_t rz, int64_t n1,
                                      int64_t r2) {
  if (rl <= 0 || n <= 0 || rx <= 0 || rz <= 0 || n1 <= 0 || r2 <= 0) return 0;
  bool ok = true;
  const long long cat = prod({rl, n, rx + rz}, ok), cat1 = prod({rx + rz, n1, r2}, ok);
  if (!ok) return 0;
  const size_t mv = tt_block_move_workspace_size(rl, n, 1, rx + rz, n1, r2);
  if (mv == 0) return 0;
  return mv + ws_bytes({cat, cat1});
}

static tt_status enrich_right_impl(int64_t rl, int64_t n, int64_t rx, int64_t rz, int64_t n1, int64_t r2,
                          double delta, int64_t max_rank, const double* x_k, const double* z_k,
                          const double* x_k1, double* x_k_out, double* x_k1_out, int64_t* s_out,
                          void* workspace, size_t workspace_bytes, void* stream, int64_t* s_dev) {
  if (rl <= 0 || n <= 0 || rx <= 0 || rz <= 0 || n1 <= 0 || r2 <= 0)
    return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  if (!x_k || !z_k || !x_k1 || !x_k_out || !x_k1_out || !s_out)
    return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  for (const void* o : {(const void*)x_k_out, (const void*)x_k1_out})
    if (same(o, x_k) || same(o, z_k) || same(o, x_k1))
      return fail(TT_ERR_ALIASING, "an output aliases an input");
  const size_t need = tt_enrich_right_workspace_size(rl, n, rx, rz, n1, r2);
  if (need == 0) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  const size_t mv = tt_block_move_workspace_size(rl, n, 1, rx + rz, n1, r2);
  char* base = static_cast<char*>(workspace);
  Carver c{base + mv, workspace_bytes - mv};
  const long long r = rx + rz;
  double* cat = c.take(rl * n * r);
  double* cat1 = c.take(r * n1 * r2);
  if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long tot = rl * n * r + r * n1 * r2;
  enrich_concat_kernel<<<(unsigned)std::min<long long>(4096, (tot + 255) / 256), 256, 0, s>>>(
      x_k, z_k, x_k1, cat, cat1, rl * n, rx, rz, n1 * r2);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "tt_enrich_right");
  const int64_t launches = g_launches;
  tt_status st = s_dev ? tt_block_move_right_async(rl, n, 1, r, n1, r2, delta, max_rank, cat, cat1,
                                                   x_k_out, x_k1_out, s_out, s_dev, base, mv, stream)
                       : tt_block_move_right(rl, n, 1, r, n1, r2, delta, max_rank, cat, cat1,
                                             x_k_out, x_k1_out, s_out, base, mv, stream);
  g_launches += launches;
  g_launches_last = g_launches;
  return st;
}
tt_status tt_enrich_right(int64_t rl, int64_t n, int64_t rx, int64_t rz, int64_t n1, int64_t r2,
                          double delta, int64_t max_rank, const double* x_k, const double* z_k,
                          const double* x_k1, double* x_k_out, double* x_k1_out, int64_t* s_out,
                          void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  return enrich_right_impl(rl, n, rx, rz, n1, r2, delta, max_rank, x_k, z_k, x_k1, x_k_out,
                           x_k1_out, s_out, workspace, workspace_bytes, stream, nullptr);
}
tt_status tt_enrich_right_async(int64_t rl, int64_t n, int64_t rx, int64_t rz, int64_t n1,
                                int64_t r2, double delta, int64_t max_rank, const double* x_k,
                                const double* z_k, const double* x_k1, double* x_k_out,
                                double* x_k1_out, int64_t* s_storage, int64_t* s_dev,
                                void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  if (!s_dev) return fail(TT_ERR_NULL_POINTER, "s_dev is NULL");
  return enrich_right_impl(rl, n, rx, rz, n1, r2, delta, max_rank, x_k, z_k, x_k1, x_k_out,
                           x_k1_out, s_storage, workspace, workspace_bytes, stream, s_dev);
}

// ---- projected KKT block system action -----------------------------
static bool block_ws(int64_t rl, int64_t n, int64_t rr, int64_t nops, const int64_t* Rl,
                     const int64_t* Rr, long long& t1, long long& t2, long long& ah, long long& pe,
                     long long& vec) {
  t1 = t2 = ah = pe = 0;
  bool ok = true;
  for (int64_t o = 0; o < nops; ++o) {
    Dims d{rl, n, rr, Rl[o], Rr[o]};
    long long a, b, c, e;
    if (!dims_valid(d) || !matvec_ws_elems(d, 1, a, b, c, e)) return false;
    t1 = std::max(t1, a);
    t2 = std::max(t2, b);
    ah = std::max(ah, c);
    pe = std::max(pe, e);
  }
  vec = prod({rl, n, rr}, ok);
  return ok;
}

size_t tt_block_local_matvec_workspace_size(int64_t rl, int64_t n, int64_t rr, int64_t nops,
                                            const int64_t* Rl, const int64_t* Rr) {
  if (nops <= 0 || !Rl || !Rr) return 0;
  long long t1, t2, ah, pe, vec;
  if (!block_ws(rl, n, rr, nops, Rl, Rr, t1, t2, ah, pe, vec)) return 0;
  // one matvec lane per pool stream: the terms' matvecs run concurrently
  return (size_t)kPoolStreams * ws_bytes({t1, t2, ah, pe, vec, vec, vec});
}

tt_status tt_block_local_matvec(int64_t rl, int64_t n, int64_t rr, int64_t nblocks, int64_t nops,
                                const int64_t* Rl, const int64_t* Rr, const double* const* phiL,
                                const double* const* A, const double* const* phiR,
                                int64_t nterms, const tt_block_term* terms, const double* X,
                                double* Y, void* workspace, size_t workspace_bytes,
                                void* stream) {
  CallScope scope;
  if (rl <= 0 || n <= 0 || rr <= 0 || nblocks <= 0 || nops <= 0 || nterms < 0)
    return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  if (!Rl || !Rr || !phiL || !A || !phiR || !X || !Y || (nterms > 0 && !terms))
    return fail(TT_ERR_NULL_POINTER, "NULL argument");
  for (int64_t o = 0; o < nops; ++o) {
    if (!phiL[o] || !A[o] || !phiR[o]) return fail(TT_ERR_NULL_POINTER, "NULL operator entry");
    tt_status st = check_dims(Dims{rl, n, rr, Rl[o], Rr[o]});
    if (st != TT_OK) return st;
    if (same(Y, phiL[o]) || same(Y, A[o]) || same(Y, phiR[o]))
      return fail(TT_ERR_ALIASING, "output Y aliases an operator");
  }
  if (same(Y, X)) return fail(TT_ERR_ALIASING, "output Y aliases X");
  for (int64_t t = 0; t < nterms; ++t) {
    const tt_block_term& tm = terms[t];
    if (tm.row < 0 || tm.row >= nblocks || tm.col < 0 || tm.col >= nblocks || tm.op < 0 ||
        tm.op >= nops || tm.op2 < -1 || tm.op2 >= nops)
      return fail(TT_ERR_INVALID_ARGUMENT, "term " + std::to_string(t) + " out of range");
  }
  long long t1, t2, ah, pe, vec;
  if (!block_ws(rl, n, rr, nops, Rl, Rr, t1, t2, ah, pe, vec))
    return fail(TT_ERR_OVERFLOW, "workspace overflow");
  const size_t lane_b = ws_bytes({t1, t2, ah, pe, vec, vec, vec});
  const size_t need = (size_t)kPoolStreams * lane_b;
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  // Terms are independent K = 1 matvecs (~12 GFLOP each at the config-5 interior core: stage
  // GEMMs of 2.7-4.8 GFLOP that quantise badly on 148 SMs), so they run on up to kPoolStreams
  // lanes concurrently, each with its own scratch; the accumulation Y[row] += coeff T_t stays
  // in term order per row block (each scatter waits for the previous scatter into its row:
  // deterministic and race-free).  Lanes are assigned greedily by cost (2 for a product term).
  struct Lane {
    double *T1, *T2, *Ah, *Pp, *G, *G2, *Tv;
  };
  const int lanes = (int)std::min<int64_t>(kPoolStreams, std::max<int64_t>(nterms, 1));
  std::vector<Lane> L(size_t(lanes), Lane{});
  for (int q = 0; q < lanes; ++q) {
    Carver c{static_cast<char*>(workspace) + (size_t)q * lane_b, lane_b};
    L[q].T1 = c.take(t1);
    L[q].T2 = c.take(t2);
    L[q].Ah = c.take(ah);
    L[q].Pp = c.take(pe);
    L[q].G = c.take(vec);
    L[q].G2 = c.take(vec);
    L[q].Tv = c.take(vec);
    if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long rows = rl * n;
  long long blocks = (vec + 255) / 256;
  if (blocks > 4L * num_sms()) blocks = 4L * num_sms();
  cudaError_t e = cudaMemsetAsync(Y, 0, sizeof(double) * rows * nblocks * rr, s);
  if (e != cudaSuccess) return cuda_fail(e, "tt_block_local_matvec");
  auto term = [&](const tt_block_term& tm, const Lane& ln, cudaStream_t ps) -> cudaError_t {
    gather_col_kernel<<<(unsigned)blocks, 256, 0, ps>>>(X, ln.G, rows, (int)nblocks, (int)rr,
                                                        (int)tm.col);
    ++g_launches;
    const double* in = ln.G;
    cudaError_t r = cudaSuccess;
    if (tm.op2 >= 0) {
      const Dims d2{rl, n, rr, Rl[tm.op2], Rr[tm.op2]};
      r = enqueue_matvec(d2, 1, phiL[tm.op2], A[tm.op2], phiR[tm.op2], ln.G, ln.G2, ln.T1, ln.T2,
                         ln.Ah, ln.Pp, pe, ps);
      in = ln.G2;
    }
    if (r != cudaSuccess) return r;
    const Dims d1{rl, n, rr, Rl[tm.op], Rr[tm.op]};
    return enqueue_matvec(d1, 1, phiL[tm.op], A[tm.op], phiR[tm.op], in, ln.Tv, ln.T1, ln.T2,
                          ln.Ah, ln.Pp, pe, ps);
  };
  auto scatter = [&](const tt_block_term& tm, const Lane& ln, cudaStream_t ps) -> cudaError_t {
    scatter_add_col_kernel<<<(unsigned)blocks, 256, 0, ps>>>(ln.Tv, Y, rows, (int)nblocks,
                                                             (int)rr, (int)tm.row, tm.coeff);
    ++g_launches;
    return cudaGetLastError();
  };
  if (lanes <= 1 || (g_dbg_flags & 8)) {   // one lane on the caller's stream (debug bit 3: A/B)
    for (int64_t t = 0; t < nterms && e == cudaSuccess; ++t) {
      e = term(terms[t], L[0], s);
      if (e == cudaSuccess) e = scatter(terms[t], L[0], s);
    }
    if (e != cudaSuccess) return cuda_fail(e, "tt_block_local_matvec");
    return TT_OK;
  }
  if ((e = pool_init(size_t(nterms + kPoolStreams + 2))) != cudaSuccess) return cuda_fail(e, "pool");
  cudaEvent_t* ev = g_res.pool.ev.data();   // ev[t]: term t's scatter done; ev[nterms + q]: joins
  for (int q = 0; q < lanes && e == cudaSuccess; ++q) e = stream_dep(s, g_res.pool.s[q]);
  std::vector<int> cost(size_t(lanes), 0);
  std::vector<int64_t> last_in_row(size_t(nblocks), -1);
  for (int64_t t = 0; t < nterms && e == cudaSuccess; ++t) {
    const tt_block_term& tm = terms[t];
    int q = 0;
    for (int i = 1; i < lanes; ++i)
      if (cost[size_t(i)] < cost[size_t(q)]) q = i;
    cost[size_t(q)] += tm.op2 >= 0 ? 2 : 1;
    cudaStream_t ps = g_res.pool.s[q];
    if ((e = term(tm, L[size_t(q)], ps)) != cudaSuccess) break;
    const int64_t prev = last_in_row[size_t(tm.row)];
    if (prev >= 0 && (e = cudaStreamWaitEvent(ps, ev[prev], 0)) != cudaSuccess) break;
    if ((e = scatter(tm, L[size_t(q)], ps)) != cudaSuccess) break;
    if ((e = cudaEventRecord(ev[t], ps)) != cudaSuccess) break;
    last_in_row[size_t(tm.row)] = t;
  }
  for (int q = 0; q < lanes && e == cudaSuccess; ++q)
    if ((e = cudaEventRecord(ev[nterms + q], g_res.pool.s[q])) == cudaSuccess)
      e = cudaStreamWaitEvent(s, ev[nterms + q], 0);
  if (e != cudaSuccess) return cuda_fail(e, "tt_block_local_matvec");
  return TT_OK;
}

// ---- two-site local matvec ------------------------------------------
size_t tt_local_matvec_two_site_workspace_size(int64_t rl, int64_t n1, int64_t n2, int64_t rr,
                                               int64_t Rl, int64_t Rm, int64_t Rr, int64_t nvec) {
  if (n1 <= 0 || n2 <= 0 || Rm <= 0 || nvec <= 0) return 0;
  Dims d{rl, n1 * n2, rr, Rl, Rr};
  long long t1, t2, ah, pe;
  if (!dims_valid(d) || !matvec_ws_elems(d, nvec, t1, t2, ah, pe)) return 0;
  return ws_bytes({t1, t2, ah, pe, d.al * d.n * d.n * d.be});
}

tt_status tt_local_matvec_two_site(int64_t rl, int64_t n1, int64_t n2, int64_t rr, int64_t Rl,
                                   int64_t Rm, int64_t Rr, int64_t nvec, const double* phiL,
                                   const double* A1, const double* A2, const double* phiR,
                                   const double* W, double* Y, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  CallScope scope;
  if (n1 <= 0 || n2 <= 0 || Rm <= 0 || nvec <= 0)
    return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  bool ok = true;
  const long long N = prod({n1, n2}, ok);
  if (!ok) return fail(TT_ERR_OVERFLOW, "extent product overflows");
  Dims d{rl, N, rr, Rl, Rr};
  tt_status st = check_dims(d);
  if (st != TT_OK) return st;
  if (!phiL || !A1 || !A2 || !phiR || !W || !Y) return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  if (same(Y, phiL) || same(Y, A1) || same(Y, A2) || same(Y, phiR) || same(Y, W))
    return fail(TT_ERR_ALIASING, "output Y aliases an input");
  long long t1, t2, ah, pe;
  if (!matvec_ws_elems(d, nvec, t1, t2, ah, pe)) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  const long long a12 = d.al * d.n * d.n * d.be;
  const size_t need = ws_bytes({t1, t2, ah, pe, a12});
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  Carver c{static_cast<char*>(workspace), workspace_bytes};
  double* T1 = c.take(t1);
  double* T2 = c.take(t2);
  double* Ah = c.take(ah);
  double* Pp = c.take(pe);
  double* A12 = c.take(a12);
  if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  long long blocks = (a12 + 255) / 256;
  if (blocks > 2048) blocks = 2048;
  g_stage = TT_ST_PERM;
  const long long tr = trace_begin(0, a12, 0, 0, s);
  merge_cores_kernel<<<(unsigned)blocks, 256, 0, s>>>(A1, A2, A12, Rl, n1, n2, Rm, Rr);
  trace_end(tr, s);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = enqueue_matvec(d, nvec, phiL, A12, phiR, W, Y, T1, T2, Ah, Pp, pe, s);
  if (e != cudaSuccess) return cuda_fail(e, "tt_local_matvec_two_site");
  return TT_OK;
}

// ---- local GMRES --------------------------------------------------
size_t tt_local_gmres_workspace_size(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr,
                                     int64_t nvec, int64_t m, int64_t k_aug) {
  Dims d{rl, n, rr, Rl, Rr};
  long long t1, t2, ah, pe;
  GmresWs gw;
  if (!dims_valid(d) || nvec <= 0 || nvec > 64 || m <= 0 || k_aug < 0 ||
      !matvec_ws_elems(d, nvec, t1, t2, ah, pe) || !gmres_ws_elems(d, nvec, m + k_aug, gw, k_aug))
    return 0;
  return ws_bytes({t1, t2, ah, pe, gw.basis, gw.w, gw.part, gw.small});
}

tt_status tt_local_gmres(int64_t rl, int64_t n, int64_t rr, int64_t Rl, int64_t Rr, int64_t nvec,
                         int64_t m, int64_t k_aug, int64_t cycles, double tol, const double* phiL,
                         const double* A, const double* phiR, const double* F, double* X,
                         double* rel_res, int64_t* iters, void* workspace,
                         size_t workspace_bytes, void* stream) {
  CallScope scope;
  Dims d{rl, n, rr, Rl, Rr};
  tt_status st = check_dims(d);
  if (st != TT_OK) return st;
  if (nvec <= 0 || nvec > 64) return fail(TT_ERR_INVALID_ARGUMENT, "nvec must be in [1, 64]");
  if (m <= 0 || m > 512 || k_aug < 0 || k_aug > 64 || cycles < 0 || !(tol >= 0.0))
    return fail(TT_ERR_INVALID_ARGUMENT,
                "need 0 < m <= 512, 0 <= k_aug <= 64, cycles >= 0, tol >= 0");
  if (!phiL || !A || !phiR || !F || !X || !rel_res || !iters)
    return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  for (const void* o : {(const void*)X, (const void*)rel_res, (const void*)iters})
    for (const void* i : {(const void*)phiL, (const void*)A, (const void*)phiR, (const void*)F})
      if (o == i) return fail(TT_ERR_ALIASING, "an output aliases an input");
  if ((const void*)X == (const void*)rel_res || (const void*)X == (const void*)iters ||
      (const void*)rel_res == (const void*)iters)
    return fail(TT_ERR_ALIASING, "two outputs alias");
  const size_t need = tt_local_gmres_workspace_size(rl, n, rr, Rl, Rr, nvec, m, k_aug);
  if (need == 0) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  cudaError_t e = enqueue_gmres(d, nvec, m, k_aug, cycles, tol, phiL, A, phiR, F, X, rel_res,
                                reinterpret_cast<long long*>(iters), workspace, workspace_bytes,
                                static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tt_local_gmres");
  return TT_OK;
}

// ---- Petrov-Galerkin local operations (bra != ket) and AMEn enrichment ---------------------
static tt_status check_pg(const DimsPG& d) {
  if (!dims_pg_valid(d)) return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  long long t1, t2, ah, pe;
  if (!pg_ws_elems(d, 1, t1, t2, ah, pe)) return fail(TT_ERR_OVERFLOW, "extent product overflows");
  return TT_OK;
}

size_t tt_pg_workspace_size(int64_t rl_bra, int64_t rl, int64_t n, int64_t rr_bra, int64_t rr,
                            int64_t Rl, int64_t Rr, int64_t nvec) {
  DimsPG d{rl_bra, rl, n, rr_bra, rr, Rl, Rr};
  long long t1, t2, ah, pe;
  if (!dims_pg_valid(d) || nvec <= 0 || !pg_ws_elems(d, nvec, t1, t2, ah, pe)) return 0;
  return ws_bytes({t1, t2, ah, pe});
}

#define TT_PG_CARVE()                                                                      \
  long long t1, t2, ah, pe;                                                                \
  if (!pg_ws_elems(d, K, t1, t2, ah, pe)) return fail(TT_ERR_OVERFLOW, "workspace overflow"); \
  const size_t need = ws_bytes({t1, t2, ah, pe});                                          \
  if (!workspace || workspace_bytes < need)                                                \
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes"); \
  Carver c{static_cast<char*>(workspace), workspace_bytes};                                \
  double* T1 = c.take(t1);                                                                 \
  double* T2 = c.take(t2);                                                                 \
  double* Ah = c.take(ah);                                                                 \
  double* Pp = c.take(pe);                                                                 \
  if (!c.ok) return fail(TT_ERR_WORKSPACE, "workspace too small after alignment");

tt_status tt_local_matvec_pg(int64_t rl_bra, int64_t rl, int64_t n, int64_t rr_bra, int64_t rr,
                             int64_t Rl, int64_t Rr, int64_t nvec, const double* phiL,
                             const double* A, const double* phiR, const double* X, double* Y,
                             void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  DimsPG d{rl_bra, rl, n, rr_bra, rr, Rl, Rr};
  tt_status st = check_pg(d);
  if (st != TT_OK) return st;
  if (nvec <= 0) return fail(TT_ERR_INVALID_ARGUMENT, "nvec must be positive");
  if (!phiL || !A || !phiR || !X || !Y) return fail(TT_ERR_NULL_POINTER, "NULL tensor pointer");
  if (same(Y, phiL) || same(Y, A) || same(Y, phiR) || same(Y, X))
    return fail(TT_ERR_ALIASING, "output Y aliases an input");
  const long long K = nvec;
  TT_PG_CARVE();
  cudaError_t e = enqueue_matvec_pg(d, K, phiL, A, phiR, X, Y, T1, T2, Ah, Pp, pe,
                                    static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tt_local_matvec_pg");
  return TT_OK;
}

tt_status tt_interface_left_pg(int64_t rl_bra, int64_t rl, int64_t n, int64_t rr_bra, int64_t rr,
                               int64_t Rl, int64_t Rr, const double* phiL_prev, const double* A,
                               const double* x_bra, const double* x_ket, double* phiL_next,
                               void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  DimsPG d{rl_bra, rl, n, rr_bra, rr, Rl, Rr};
  tt_status st = check_pg(d);
  if (st != TT_OK) return st;
  if (!phiL_prev || !A || !x_bra || !x_ket || !phiL_next)
    return fail(TT_ERR_NULL_POINTER, "NULL tensor pointer");
  if (same(phiL_next, phiL_prev) || same(phiL_next, A) || same(phiL_next, x_bra) ||
      same(phiL_next, x_ket))
    return fail(TT_ERR_ALIASING, "output aliases an input");
  const long long K = 1;
  TT_PG_CARVE();
  cudaError_t e = enqueue_left_pg(d, phiL_prev, A, x_bra, x_ket, phiL_next, T1, T2, Ah, Pp, pe,
                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tt_interface_left_pg");
  return TT_OK;
}

tt_status tt_interface_right_pg(int64_t rl_bra, int64_t rl, int64_t n, int64_t rr_bra, int64_t rr,
                                int64_t Rl, int64_t Rr, const double* phiR_next, const double* A,
                                const double* x_bra, const double* x_ket, double* phiR_prev,
                                void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  DimsPG d{rl_bra, rl, n, rr_bra, rr, Rl, Rr};
  tt_status st = check_pg(d);
  if (st != TT_OK) return st;
  if (!phiR_next || !A || !x_bra || !x_ket || !phiR_prev)
    return fail(TT_ERR_NULL_POINTER, "NULL tensor pointer");
  if (same(phiR_prev, phiR_next) || same(phiR_prev, A) || same(phiR_prev, x_bra) ||
      same(phiR_prev, x_ket))
    return fail(TT_ERR_ALIASING, "output aliases an input");
  const long long K = 1;
  TT_PG_CARVE();
  cudaError_t e = enqueue_right_pg(d, phiR_next, A, x_bra, x_ket, phiR_prev, T1, T2, Ah, Pp, pe,
                                   static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tt_interface_right_pg");
  return TT_OK;
}
#undef TT_PG_CARVE

// ---- LOBPCG ---------------------------------------------------------
size_t tt_local_lobpcg_workspace_size(int64_t rl, int64_t n, int64_t rr, int64_t RlA, int64_t RrA,
                                      int64_t RlB, int64_t RrB, int64_t nb) {
  Dims dA{rl, n, rr, RlA, RrA};
  const bool has_B = RlB > 0 || RrB > 0;
  Dims dB{rl, n, rr, has_B ? RlB : 1, has_B ? RrB : 1};
  if (!dims_valid(dA) || !dims_valid(dB) || nb <= 0 || nb > kLobMaxNb) return 0;
  long long t1a, t2a, aha, pea, t1b = 0, t2b = 0, ahb = 0, peb = 0;
  if (!matvec_ws_elems(dA, nb, t1a, t2a, aha, pea)) return 0;
  if (has_B && !matvec_ws_elems(dB, nb, t1b, t2b, ahb, peb)) return 0;
  LobWs lw;
  if (!lob_ws_elems(dA, nb, lw)) return 0;
  return ws_bytes({std::max(t1a, t1b), std::max(t2a, t2b), std::max(pea, peb), aha, ahb, lw.blocks,
                   lw.part, lw.gpart, lw.G, lw.Y, lw.small});
}

tt_status tt_local_lobpcg(int64_t rl, int64_t n, int64_t rr, int64_t RlA, int64_t RrA,
                          int64_t RlB, int64_t RrB, int64_t nb, int64_t maxiter,
                          int64_t refresh, double tol, const double* phiLA, const double* AA, const double* phiRA,
                          const double* phiLB, const double* AB, const double* phiRB, double* X,
                          double* lam, double* res, int64_t* iters, double* step,
                          void* workspace, size_t workspace_bytes, void* stream) {
  CallScope scope;
  const bool has_B = phiLB || AB || phiRB;
  if (has_B && (!phiLB || !AB || !phiRB))
    return fail(TT_ERR_NULL_POINTER, "operator B needs all of phiL_B, A_B, phiR_B (or none: B = I)");
  Dims dA{rl, n, rr, RlA, RrA};
  tt_status st = check_dims(dA);
  if (st != TT_OK) return st;
  Dims dB{rl, n, rr, has_B ? RlB : 1, has_B ? RrB : 1};
  if ((st = check_dims(dB)) != TT_OK) return st;
  if (nb <= 0 || nb > kLobMaxNb) return fail(TT_ERR_INVALID_ARGUMENT, "nb must be in [1, 32]");
  if (nb > rl * n * rr) return fail(TT_ERR_INVALID_ARGUMENT, "nb exceeds the local dimension");
  if (maxiter < 0 || refresh < 0 || !(tol >= 0.0))
    return fail(TT_ERR_INVALID_ARGUMENT, "need maxiter >= 0, refresh >= 0, tol >= 0");
  if (!phiLA || !AA || !phiRA || !X || !lam || !res || !iters)
    return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  const void* outs[] = {X, lam, res, iters, step};
  const void* ins[] = {phiLA, AA, phiRA, phiLB, AB, phiRB};
  for (const void* o : outs) {
    for (const void* i : ins)
      if (same(o, i)) return fail(TT_ERR_ALIASING, "an output aliases an input");
    for (const void* o2 : outs)
      if (o != o2 && same(o, o2)) return fail(TT_ERR_ALIASING, "two outputs alias");
  }
  const size_t need = tt_local_lobpcg_workspace_size(rl, n, rr, RlA, RrA, has_B ? RlB : 0,
                                                     has_B ? RrB : 0, nb);
  if (need == 0) return fail(TT_ERR_OVERFLOW, "workspace overflow");
  if (!workspace || workspace_bytes < need)
    return fail(TT_ERR_WORKSPACE, "workspace NULL or smaller than " + std::to_string(need) + " bytes");
  cudaError_t e = enqueue_lobpcg(dA, dB, has_B, nb, maxiter, refresh, tol, phiLA, AA, phiRA, phiLB, AB,
                                 phiRB, X, lam, res, reinterpret_cast<long long*>(iters), step,
                                 workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tt_local_lobpcg");
  return TT_OK;
}

tt_status tt_merge_operator_cores(int64_t Rl, int64_t n1, int64_t n2, int64_t Rm, int64_t Rr,
                                  const double* A1, const double* A2, double* A12, void* stream) {
  CallScope scope;
  if (Rl <= 0 || n1 <= 0 || n2 <= 0 || Rm <= 0 || Rr <= 0)
    return fail(TT_ERR_INVALID_ARGUMENT, "extents must be positive");
  bool ok = true;
  const long long total = prod({Rl, n1, n2, n1, n2, Rr}, ok);
  prod({Rl, n1, n1, Rm}, ok);
  prod({Rm, n2, n2, Rr}, ok);
  if (!ok) return fail(TT_ERR_OVERFLOW, "extent product overflows");
  if (!A1 || !A2 || !A12) return fail(TT_ERR_NULL_POINTER, "NULL pointer");
  if (same(A12, A1) || same(A12, A2)) return fail(TT_ERR_ALIASING, "output A12 aliases an input");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  long long blocks = (total + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  merge_cores_kernel<<<(unsigned)blocks, 256, 0, s>>>(A1, A2, A12, Rl, n1, n2, Rm, Rr);
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "tt_merge_operator_cores");
  return TT_OK;
}

}  // extern "C"
