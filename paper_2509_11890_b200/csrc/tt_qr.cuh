// tt_qr.cuh — Householder QR of an m x c core unfolding in ONE thread-block cluster (sm_100a).
//
// TT orthonormalisation (the rounding's orthonormalisation sweeps and the
// block-index move) needs M = Q R with Q orthonormal to working precision.  The Gram route
// (M^T M -> eigenvectors) squares the condition number; Householder reflections do not.  A
// config-5 interior unfolding (1024 x 256, 2 MB) is spread over the distributed shared memory of
// a 16-CTA cluster (64 rows per CTA), so every column step works on-chip:
//   step j:  sigma^2 = sum_{i>j} M[i][j]^2 and the dots of the column with the trailing ones
//            (per-CTA partials combined through DSMEM in rank
//            order, identical in every CTA), the reflector (LAPACK dlarfg convention:
//            beta = -sign(x_j) ||x||, tau = (beta - x_j) / beta, v = x / (x_j - beta), v_j = 1)
//            stored in place below the diagonal;
//            w = v^T M[j:, j+1:] (DSMEM-combined partials), M[i][col] -= tau v_i w[col].
//   then R is read off the upper triangle and Q = H_0 ... H_{k-1} [I; 0] is formed in place
//   backwards (LAPACK dorg2r order).
// One cluster barrier per reflector and per backward step; every reduction is deterministic.
// Included by tt_solvers.cu inside namespace ttint.

constexpr int kQrThreads = 512;
constexpr size_t kQrSmemMax = 220 * 1024;

struct QrArgs {
  const double* M;     // input, M[i][j] at M[i * rs + j * cs]
  long long rs, cs;
  int m, c;            // rows, columns; k = min(m, c) reflectors
  double* Q;           // output Q (m x k), Q[i][j] at Q[i * qrs + j * qcs] (may alias M)
  long long qrs, qcs;
  double* R;           // output R (k x c), row-major, zeros below the diagonal
  int rb;              // rows per CTA
};

__global__ void __launch_bounds__(kQrThreads) qr_cluster_kernel(const QrArgs p) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank(), ncl = (int)cluster.num_blocks();
  const int tid = threadIdx.x;
  const int m = p.m, c = p.c, k = min(m, c), rb = p.rb, ld = c + 1;   // odd row stride
  extern __shared__ double qsm[];
  double* A = qsm;                       // [rb][ld] this CTA's rows
  double* inbox = A + (size_t)rb * ld;   // [2][16][c + 2] partials pushed by every CTA
  double* tau = inbox + 2 * 16 * (c + 2);   // [k]
  double* wv = tau + k;                  // [c + 2] combined sums
  double* rowj = wv + (c + 2);           // [2][c] row j of the current reflector (from its owner)
  const int r0 = rank * rb;
  const int nr = max(0, min(rb, m - r0));   // rows held by this CTA
  for (int e = tid; e < nr * c; e += kQrThreads) {
    const int i = e / c, j = e - i * c;
    A[i * ld + j] = p.M[(long long)(r0 + i) * p.rs + (long long)j * p.cs];
  }
  __syncthreads();
  int red_no = 0;   // running reduction index: inbox parity red_no & 1
  // Reductions push: the thread holding a partial stores it into slot [parity][its rank][q]
  // of EVERY CTA's inbox (remote DSMEM stores, nothing to wait for), one cluster barrier
  // (release / acquire) makes them visible, and each CTA sums its inbox locally in rank order
  // (identical, deterministic results in every CTA).  Reusing a parity two reductions later
  // is safe: a CTA reads reduction t's inbox before arriving at barrier t + 1.
  auto push = [&](int par, int q, double v, int r) {   // to CTA r
    cluster.map_shared_rank(inbox, r)[(par * 16 + rank) * (c + 2) + q] = v;
  };
  auto gather = [&](int par, int n, double* out) {
    cluster.sync();
    for (int q = tid; q < n; q += kQrThreads) {
      double s = 0.0;
      for (int r = 0; r < ncl; ++r) s += inbox[(par * 16 + r) * (c + 2) + q];
      out[q] = s;
    }
    __syncthreads();
  };
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int kWarps = kQrThreads / 32;
  // Partial dots of column j with the columns [c0, c1), local rows with global index > j:
  //   s[col] = sum_i A[i][j] A[i][col]  (+ A[j][col] in the owner of row j when unit_diag),
  // pushed to slot col - c0 of every CTA's inbox.  A half-warp owns 16 consecutive columns
  // (conflict-free row reads, the A[i][j] factor a broadcast) and one row parity; the row
  // loop carries two independent accumulators and no shuffles except the final parity add.
  auto dots = [&](int par, int j, int c0, int c1, bool unit_diag) {
    const int ib1 = max(0, min(nr, j + 1 - r0));   // first local row with global index > j
    const int h = lane >> 4;
    const bool diag_here = unit_diag && j >= r0 && j < r0 + nr;
    for (int q0 = c0; q0 < c1; q0 += kWarps * 16) {
      const int col = q0 + warp * 16 + (lane & 15);
      const bool on = col < c1;
      double s0 = 0.0, s1 = 0.0;
      if (on) {
        const double* a = A + col;
        const double* x = A + j;
        int i = ib1 + h;
#pragma unroll 2
        for (; i + 2 < nr; i += 4) {
          s0 = fma(x[i * ld], a[i * ld], s0);
          s1 = fma(x[(i + 2) * ld], a[(i + 2) * ld], s1);
        }
        if (i < nr) s0 = fma(x[i * ld], a[i * ld], s0);
        if (diag_here && h == 0) s1 += a[(j - r0) * ld];
      }
      double sv = s0 + s1;
      sv += __shfl_xor_sync(0xffffffffu, sv, 16);
      if (on)
        for (int r = h; r < ncl; r += 2) push(par, col - c0, sv, r);
    }
  };
  // A[i][col] += tv w[col - wo] for col in [c0, c1): one row per warp, eight columns per lane
  // loaded before any store (the compiler cannot reorder shared-memory loads across the stores
  // of a rolled loop, which serialised the latencies)
  auto row_axpy = [&](double* row, double tv, int c0, int c1, const double* w, int wo) {
    for (int cb = c0; cb < c1; cb += 256) {
      double a[8], ww[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int col = cb + lane + 32 * u;
        a[u] = col < c1 ? row[col] : 0.0;
        ww[u] = col < c1 ? w[col - wo] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int col = cb + lane + 32 * u;
        if (col < c1) row[col] = fma(tv, ww[u], a[u]);
      }
    }
  };
  // w[col] = sum_{i >= j} v_i M[i][col] for col in [c0, c1), v_j = 1, v_i = A[i][j] below;
  // then M[i][col] -= t v_i w[col]
  auto apply_reflector = [&](int j, int c0, int c1, double t) {
    const int par = red_no++ & 1;
    const int ib = max(0, min(nr, j - r0));   // first local row with global index >= j
    dots(par, j, c0, c1, true);
    gather(par, c1 - c0, wv);
    for (int i = ib + warp; i < nr; i += kWarps) {
      const double tv = -t * ((r0 + i == j) ? 1.0 : A[i * ld + j]);
      row_axpy(A + (size_t)i * ld, tv, c0, c1, wv, c0);
    }
    __syncthreads();
  };

  // ---- factorisation ---------------------------------------------------------------------
  // ONE cluster reduction per reflector: with x = M[j:, j], every CTA pushes its partials of
  // y[q] = sum_{i > j} x_i M[i][j + q], q = 0 .. c - j - 1 (q = 0: sigma^2, the squared norm
  // below the diagonal), and the owner of row j broadcasts M[j][j:]; after the barrier each
  // CTA derives beta, tau, the scaling of v and w = v^T M[j:, j+1:] = M[j][col] + scal y[col]
  // locally (v_j = 1, v_i = scal x_i) -- the same reflector as the two-reduction form (norm,
  // then v^T M), the sums in another order.
  for (int j = 0; j < k; ++j) {
    const int owner = j / rb;
    const int par = red_no++ & 1;
    const int ib1 = max(0, min(nr, j + 1 - r0));   // first local row with global index > j
    const int ncol = c - j;
    dots(par, j, j, c, false);
    if (rank == owner) {
      const double* row = A + (size_t)(j - r0) * ld + j;
      for (int q = tid; q < ncol; q += kQrThreads) {
        const double v = row[q];
        for (int r = 0; r < ncl; ++r) cluster.map_shared_rank(rowj, r)[par * c + q] = v;
      }
    }
    gather(par, ncol, wv);
    const double* rj = rowj + par * c;
    const double sigma2 = wv[0], xj = rj[0];
    double t = 0.0, beta = xj, scal = 0.0;
    if (sigma2 > 0.0) {
      beta = -copysign(sqrt(fma(xj, xj, sigma2)), xj);
      t = (beta - xj) / beta;
      scal = 1.0 / (xj - beta);
    }
    if (tid == 0) tau[j] = t;
    for (int q = 1 + tid; q < ncol; q += kQrThreads) wv[q] = fma(scal, wv[q], rj[q]);   // w
    __syncthreads();
    for (int i = ib1 + warp; i < nr; i += kWarps) {   // rows below j: v_i = scal x_i
      const double vi = A[i * ld + j] * scal;
      if (t != 0.0) row_axpy(A + (size_t)i * ld, -t * vi, j + 1, c, wv, j);
      __syncwarp();
      if (lane == 0) A[i * ld + j] = vi;
    }
    if (rank == owner) {   // row j: v_j = 1
      double* row = A + (size_t)(j - r0) * ld;
      if (t != 0.0)
        for (int col = j + 1 + tid; col < c; col += kQrThreads) row[col] = fma(-t, wv[col - j], row[col]);
      if (tid == 0) row[j] = beta;
    }
    __syncthreads();
  }
  // ---- R: the upper triangle of rows 0..k-1 ----------------------------------------------
  for (int e = tid; e < nr * c; e += kQrThreads) {
    const int i = e / c, col = e - i * c;
    const int gi = r0 + i;
    if (gi < k) p.R[(long long)gi * c + col] = (col >= gi) ? A[i * ld + col] : 0.0;
  }
  __syncthreads();
  // ---- Q = H_0 ... H_{k-1} [I; 0], formed in place backwards (dorg2r) ---------------------
  for (int j = k - 1; j >= 0; --j) {
    if (j < k - 1) apply_reflector(j, j + 1, k, tau[j]);
    const double t = tau[j];
    for (int i = tid; i < nr; i += kQrThreads) {
      const int gi = r0 + i;
      if (gi > j) A[i * ld + j] *= -t;
      else if (gi == j) A[i * ld + j] = 1.0 - t;
      else A[i * ld + j] = 0.0;
    }
    __syncthreads();
  }
  cluster.sync();   // every CTA's remote reads are done before Q may overwrite M (aliasing)
  for (int e = tid; e < nr * k; e += kQrThreads) {
    const int i = e / k, j = e - i * k;
    p.Q[(long long)(r0 + i) * p.qrs + (long long)j * p.qcs] = A[i * ld + j];
  }
  cluster.sync();   // no CTA leaves while another may still read its shared memory
}

// cluster size for an m-row factorisation (16 where non-portable clusters are available, per
// device); 0 when the rows do not fit the cluster's shared memory
inline int qr_cluster_size(int m, int c) {
  thread_local int cl_dev[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& cl = cl_dev[dev & 63];
  if (cl == 0) {
    cl = 8;
    if (cudaFuncSetAttribute(qr_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
            cudaSuccess &&
        smem_attr((const void*)qr_cluster_kernel, (int)kQrSmemMax) == cudaSuccess) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(16);
      q.blockDim = dim3(kQrThreads);
      q.dynamicSmemBytes = kQrSmemMax;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = 16;
      a[0].val.clusterDim.y = 1;
      a[0].val.clusterDim.z = 1;
      q.attrs = a;
      q.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, qr_cluster_kernel, &q) == cudaSuccess && n > 0) cl = 16;
    }
    cudaGetLastError();
  }
  return cl;
}
inline size_t qr_smem(int m, int c, int cl) {
  const long long rb = (m + cl - 1) / cl;
  const int k = std::min(m, c);
  return sizeof(double) * (size_t)(rb * (c + 1) + 2 * 16 * (c + 2) + k + c + 2 + 2 * c);
}
inline bool qr_fits(int m, int c) {
  if (m <= 0 || c <= 0 || c > kQrThreads * 4) return false;
  return qr_smem(m, c, qr_cluster_size(m, c)) <= kQrSmemMax;
}

// Q (m x k) and R (k x c) of M; Q may alias M.  One cluster launch.
inline cudaError_t launch_qr(const QrArgs& a0, cudaStream_t s) {
  QrArgs a = a0;
  const int cl = qr_cluster_size(a.m, a.c);
  a.rb = (a.m + cl - 1) / cl;
  const size_t smem = qr_smem(a.m, a.c, cl);
  if (smem > kQrSmemMax) return cudaErrorInvalidValue;
  if (cudaError_t e = smem_attr((const void*)qr_cluster_kernel, (int)kQrSmemMax)) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl);
  cfg.blockDim = dim3(kQrThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  g_stage = TT_ST_SET;
  const long long tr = trace_begin(-3, a.m, a.c, 0, s);
  cudaError_t e = cudaLaunchKernelEx(&cfg, qr_cluster_kernel, a);
  trace_end(tr, s);
  ++g_launches;
  return e;
}

// ---- one-sided (Hestenes) Jacobi SVD of a small rows x c matrix in one cluster ------------------
// B = R of the core's QR (rows = min(m, c) <= 256, c <= 256).  Columns are owned by the CTAs
// (cpb consecutive columns each) and stay there; in every round-robin step each column meets one
// partner, and BOTH owners compute the pair's rotation from the same canonical sums
// (alpha_p = ||b_p||^2, alpha_q = ||b_q||^2, gamma = b_p . b_q, p < q, identical code and
// summation order, so identical bits), each updating only its own column of B and of the
// accumulated rotation J; the partner's columns are read through distributed shared memory from
// the previous step's buffer (double-buffered, one cluster barrier per step).  Relative accuracy
// of the singular values does not depend on the condition number (Demmel & Veselic 1992): there
// is no squared-condition floor.  Output: B J (columns u_j sigma_j), J, sigma_j = ||(B J)_j||.
constexpr int kSvdMaxC = 256, kSvdMaxRows = 256, kSvdMaxSweeps = 60;
struct SvdArgs {
  const double* B;   // rows x c, row-major (bt = 0) or column-major (bt = 1)
  int rows, c, cpb;  // columns per CTA
  int bt;
  double* BJ;        // rows x c row-major (output)
  double* J;         // c x c row-major (output)
  double* sigma;     // c (output)
  int* sweeps;       // (output) sweeps run
};

__global__ void __launch_bounds__(kQrThreads) svd_jacobi_cluster_kernel(const SvdArgs p) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank(), ncl = (int)cluster.num_blocks();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kWarps = kQrThreads / 32;
  const int rows = p.rows, c = p.c, cpb = p.cpb, P = (c + 1) & ~1;
  extern __shared__ double ssm[];
  // [2 buffers][cpb columns][rows] of B, then of J (columns contiguous)
  double* Bb = ssm;
  double* Jb = Bb + 2 * (size_t)cpb * rows;
  int* partner = reinterpret_cast<int*>(Jb + 2 * (size_t)cpb * c);   // [P]
  __shared__ double offmax[16];
  __shared__ double sweep_off;
  const int j0 = rank * cpb;
  const int nown = max(0, min(cpb, c - j0));
  for (int e = tid; e < nown * rows; e += kQrThreads) {
    const int lj = e / rows, i = e - lj * rows;
    Bb[lj * rows + i] = p.bt ? p.B[(long long)(j0 + lj) * rows + i] : p.B[(long long)i * c + j0 + lj];
  }
  for (int e = tid; e < nown * c; e += kQrThreads) {
    const int lj = e / c, i = e - lj * c;
    Jb[lj * c + i] = (i == j0 + lj) ? 1.0 : 0.0;
  }
  cluster.sync();
  const double tol = 1e-15 * rows;
  int cur = 0, sw = 0;
  for (; sw < kSvdMaxSweeps; ++sw) {
    double my_off = 0.0;
    for (int step = 0; step < P - 1; ++step) {
      for (int k = tid; k < P / 2; k += kQrThreads) {   // the step's pairs (chess tournament)
        int a = (k == 0) ? 0 : 1 + (k - 1 + step) % (P - 1);
        int b = 1 + (P - 2 - k + step) % (P - 1);
        partner[a] = b;
        partner[b] = a;
      }
      __syncthreads();
      const double* Bc = Bb + (size_t)cur * cpb * rows;
      const double* Jc = Jb + (size_t)cur * cpb * c;
      double* Bn = Bb + (size_t)(cur ^ 1) * cpb * rows;
      double* Jn = Jb + (size_t)(cur ^ 1) * cpb * c;
      for (int lj = warp; lj < nown; lj += kWarps) {
        const int j = j0 + lj, q = partner[j];
        const double* bj = Bc + lj * rows;
        const double* jj = Jc + lj * c;
        if (q >= c) {   // dummy partner (odd c): unchanged
          for (int i = lane; i < rows; i += 32) Bn[lj * rows + i] = bj[i];
          for (int i = lane; i < c; i += 32) Jn[lj * c + i] = jj[i];
          continue;
        }
        const int oq = q / cpb, lq = q - oq * cpb;
        const double* bq = cluster.map_shared_rank(Bb, oq) + (size_t)cur * cpb * rows + lq * rows;
        const double* jq = cluster.map_shared_rank(Jb, oq) + (size_t)cur * cpb * c + lq * c;
        const bool lo = j < q;   // canonical pair (p, q) = (min, max)
        // both columns of B and of J (own: local, partner: DSMEM) go into registers in ONE
        // round of loads -- rows, c <= 256, eight per lane -- and serve the sums and both
        // updates; loops that re-read the partner between stores paid its remote latency
        // once per 32 rows
        double bo[8], bp[8], jo[8], jp[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = lane + 32 * u;
          bo[u] = i < rows ? bj[i] : 0.0;
          bp[u] = i < rows ? bq[i] : 0.0;
          jo[u] = i < c ? jj[i] : 0.0;
          jp[u] = i < c ? jq[i] : 0.0;
        }
        double sp = 0.0, sq = 0.0, g = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {   // same order as a lane-strided loop (zeros beyond rows)
          const double x = lo ? bo[u] : bp[u], y = lo ? bp[u] : bo[u];
          sp = fma(x, x, sp);
          sq = fma(y, y, sq);
          g = fma(x, y, g);
        }
        for (int o = 16; o > 0; o >>= 1) {
          sp += __shfl_xor_sync(0xffffffffu, sp, o);
          sq += __shfl_xor_sync(0xffffffffu, sq, o);
          g += __shfl_xor_sync(0xffffffffu, g, o);
        }
        double cs = 1.0, sn = 0.0;
        const double pq = sp * sq;
        if (pq > 0.0 && g * g > (tol * tol) * pq) {
          // rotation from two reciprocal square roots (jb2_rotation, tt_round.cuh): the same
          // angle as zeta = (sq - sp) / 2g, t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2))
          jb2_rotation(sp, sq, g, cs, sn);
          my_off = fmax(my_off, fabs(g) * rsqrt(pq));
        }
        // [b_p', b_q'] = [b_p, b_q] [[cs, sn], [-sn, cs]]
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = lane + 32 * u;
          const double x = lo ? bo[u] : bp[u], y = lo ? bp[u] : bo[u];
          if (i < rows) Bn[lj * rows + i] = lo ? fma(-sn, y, cs * x) : fma(sn, x, cs * y);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = lane + 32 * u;
          const double x = lo ? jo[u] : jp[u], y = lo ? jp[u] : jo[u];
          if (i < c) Jn[lj * c + i] = lo ? fma(-sn, y, cs * x) : fma(sn, x, cs * y);
        }
      }
      cluster.sync();   // every read of the cur buffers is done; nxt is complete
      cur ^= 1;
    }
    // convergence: the largest rotated pair of the sweep, over the cluster (rank order)
    for (int o = 16; o > 0; o >>= 1) my_off = fmax(my_off, __shfl_xor_sync(0xffffffffu, my_off, o));
    __shared__ double wmax[kQrThreads / 32];
    if (lane == 0) wmax[warp] = my_off;
    __syncthreads();
    if (tid == 0) {
      double mx = 0.0;
      for (int w = 0; w < kWarps; ++w) mx = fmax(mx, wmax[w]);
      for (int r = 0; r < ncl; ++r) cluster.map_shared_rank(offmax, r)[rank] = mx;
    }
    cluster.sync();
    if (tid == 0) {
      double mx = 0.0;
      for (int r = 0; r < ncl; ++r) mx = fmax(mx, offmax[r]);
      sweep_off = mx;
    }
    __syncthreads();
    if (sweep_off == 0.0) break;   // no rotation in the whole sweep: converged
  }
  const double* Bc = Bb + (size_t)cur * cpb * rows;
  const double* Jc = Jb + (size_t)cur * cpb * c;
  for (int lj = warp; lj < nown; lj += kWarps) {
    double s = 0.0;
    for (int i = lane; i < rows; i += 32) s = fma(Bc[lj * rows + i], Bc[lj * rows + i], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) p.sigma[j0 + lj] = sqrt(s);
  }
  for (int e = tid; e < nown * rows; e += kQrThreads) {
    const int lj = e / rows, i = e - lj * rows;
    p.BJ[(long long)i * c + j0 + lj] = Bc[lj * rows + i];
  }
  for (int e = tid; e < nown * c; e += kQrThreads) {
    const int lj = e / c, i = e - lj * c;
    p.J[(long long)i * c + j0 + lj] = Jc[lj * c + i];
  }
  if (rank == 0 && tid == 0 && p.sweeps) *p.sweeps = sw;
  cluster.sync();
}

inline size_t svd_smem(int rows, int c, int cpb) {
  return sizeof(double) * (size_t)(2 * cpb * rows + 2 * cpb * c) + sizeof(int) * (size_t)(c + 2);
}
inline bool svd_fits(int rows, int c) {
  if (rows <= 0 || c <= 0 || rows > kSvdMaxRows || c > kSvdMaxC) return false;
  const int cl = qr_cluster_size(rows, c);
  const int cpb = (c + cl - 1) / cl;
  return svd_smem(rows, c, cpb) <= kQrSmemMax;
}
inline cudaError_t launch_svd(SvdArgs a, cudaStream_t s) {
  const int cl = qr_cluster_size(a.rows, a.c);
  a.cpb = (a.c + cl - 1) / cl;
  const size_t smem = svd_smem(a.rows, a.c, a.cpb);
  if (smem > kQrSmemMax) return cudaErrorInvalidValue;
  if (cudaError_t e = smem_attr((const void*)svd_jacobi_cluster_kernel, (int)kQrSmemMax)) return e;
  cudaFuncSetAttribute(svd_jacobi_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl);
  cfg.blockDim = dim3(kQrThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  g_stage = TT_ST_SET;
  const long long tr = trace_begin(-5, a.rows, a.c, 0, s);
  cudaError_t e = cudaLaunchKernelEx(&cfg, svd_jacobi_cluster_kernel, a);
  trace_end(tr, s);
  ++g_launches;
  return e;
}
